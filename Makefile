# Builds every native artefact in-tree (the .so files travel to the GPU box
# with the gpurun snapshot; they are git-ignored).
#   paper_2106_12836_b200/libsait_b200.so   CUDA kernels + C ABI (include/sait_c.h)
#   paper_2106_12836_b200/libsaitprec_b200.so  drop-in C++ saitprec:: API over the C ABI
#   oracle/liboracle.so, oracle/_ref/libsaitref.so  test oracle (see oracle/Makefile)
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2106_12836_b200
CSRC := $(PKG)/csrc
BUILD := build

# sm_100a only.  --fmad=false + explicit __dmul_rn/__dadd_rn: every product is
# rounded before it is added, as in the reference (no FMA contraction).
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC,-ffp-contract=off,-Wall,-fopenmp \
           -Iinclude -I$(CSRC) -Xptxas -warn-spills
CXXFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -Wall -Iinclude -I/usr/local/cuda/include

CU_SRCS := csr_ops split spgemm spmv sell blas solvers trisolve ilu aux_ops cap capi
CU_OBJS := $(addprefix $(BUILD)/,$(addsuffix .o,$(CU_SRCS)))
HOST_OBJS := $(BUILD)/host_inputs.o $(BUILD)/host_mm.o
HEADERS := include/sait_c.h $(wildcard $(CSRC)/*.cuh)

SHIM_SRCS := $(wildcard $(CSRC)/shim/*.cpp)
SHIM_HDRS := $(wildcard include/saitprec/*.hpp)

all: $(PKG)/libsait_b200.so shim $(BUILD)/shim_check oracle checked

$(BUILD)/%.o: $(CSRC)/%.cu $(HEADERS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(BUILD)/host_%.o: $(CSRC)/host_%.cpp include/sait_c.h
	@mkdir -p $(BUILD)
	g++ $(CXXFLAGS) -O3 -fopenmp -c -o $@ $<

$(PKG)/libsait_b200.so: $(CU_OBJS) $(HOST_OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(CU_OBJS) $(HOST_OBJS) -cudart static -lgomp

shim: $(PKG)/libsaitprec_b200.so

$(PKG)/libsaitprec_b200.so: $(SHIM_SRCS) $(SHIM_HDRS) $(PKG)/libsait_b200.so include/sait_c.h
	@if [ -n "$(SHIM_SRCS)" ]; then \
	  g++ $(CXXFLAGS) -shared -o $@ $(SHIM_SRCS) -L$(PKG) -lsait_b200 -Wl,-rpath,'$$ORIGIN'; \
	fi

# a program written against the reference's saitprec:: headers, linked to the shim
$(BUILD)/shim_check: tests/cpp/shim_check.cpp $(PKG)/libsaitprec_b200.so $(SHIM_HDRS)
	@mkdir -p $(BUILD)
	g++ $(CXXFLAGS) -o $@ $< -L$(PKG) -lsaitprec_b200 -lsait_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# the bounds-checked build (SAIT_DEVICE_CHECKS: device index range checks
# that print and trap), loaded with SAIT_CHECKED=1 -- the stand-in for
# compute-sanitizer on a pool that does not allow it (tools/sanitize.py)
CHECKED := $(PKG)/checked
checked: $(CHECKED)/libsait_b200.so

$(BUILD)/checked/%.o: $(CSRC)/%.cu $(HEADERS)
	@mkdir -p $(BUILD)/checked
	$(NVCC) $(NVFLAGS) -DSAIT_DEVICE_CHECKS -c -o $@ $<

$(CHECKED)/libsait_b200.so: $(addprefix $(BUILD)/checked/,$(addsuffix .o,$(CU_SRCS))) $(HOST_OBJS)
	@mkdir -p $(CHECKED)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $^ -cudart static -lgomp

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(BUILD) $(PKG)/*.so $(CHECKED)
	$(MAKE) -C oracle clean

.PHONY: all shim oracle clean checked
