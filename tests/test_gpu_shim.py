"""The drop-in C++ API: a program written against the reference's saitprec::
headers (tests/cpp/shim_check.cpp), linked against libsaitprec_b200.so, must
reproduce the reference's own outputs bitwise (golden fixtures made by the
compiled reference) and raise the reference's exception types/messages."""
import os
import struct
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden_csr
from helpers import bitwise_equal

pytestmark = pytest.mark.gpu


def read_dump(path):
    out = {}
    with open(path, "rb") as f:
        data = f.read()
    p = 0
    while p < len(data):
        (l,) = struct.unpack_from("<i", data, p)
        p += 4
        name = data[p : p + l].decode()
        p += l
        t = chr(data[p])
        p += 1
        (n,) = struct.unpack_from("<q", data, p)
        p += 8
        dt = np.float64 if t == "d" else np.int64
        out[name] = np.frombuffer(data, dtype=dt, count=n, offset=p).copy()
        p += 8 * n
    return out


@pytest.fixture(scope="module")
def dump(tmp_path_factory):
    exe = os.path.join(ROOT, "build", "shim_check")
    assert os.path.exists(exe), "build/shim_check missing (make)"
    path = str(tmp_path_factory.mktemp("shim") / "out.bin")
    r = subprocess.run([exe, path], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    return read_dump(path)


def csr_eq(d, name, g, gname):
    ref = golden_csr(g, gname)
    return (
        np.array_equal(d[name + "/row_ptr"], ref.row_ptr)
        and np.array_equal(d[name + "/col_idx"], ref.col_idx)
        and bitwise_equal(d[name + "/values"], ref.values)
    )


def test_shim_matches_reference_golden(dump, golden):
    assert csr_eq(dump, "A", golden, "c1/A")
    assert csr_eq(dump, "ML", golden, "c1/ML")
    assert csr_eq(dump, "MU", golden, "c1/MU")
    assert bitwise_equal(dump["z"], golden["c1/z"])
    assert dump["pair_nnz"][0] == 2 * 51215
    assert bitwise_equal(dump["exact_z"], golden["c1/z_exact"])
    assert dump["exact_nnz"][0] == golden_csr(golden, "c1/L").nnz + golden_csr(golden, "c1/U").nnz
    assert bitwise_equal(dump["jacobi3_z"], golden["c1/z_jacobi3"])


def test_shim_builders_and_kernels_match_oracle(dump, golden, port):
    from oracle import oracle as O

    L, U = golden_csr(golden, "c1/L"), golden_csr(golden, "c1/U")

    def eq(name, m):
        return (
            np.array_equal(dump[name + "/row_ptr"], m.row_ptr)
            and np.array_equal(dump[name + "/col_idx"], m.col_idx)
            and (m.values is None or bitwise_equal(dump[name + "/values"], m.values))
        )

    assert eq("pat_2_3", port.sait_pat(L, True, 2, 3))
    assert eq("cap", port.sait_thr_cap(U, False, 1e-2, 4, 1.5))
    assert eq("patcap_2", port.sait_pat_capture_pattern(L, True, 2))
    assert eq("spgemm", port.spgemm(L, U))
    assert eq("transpose", port.transpose(golden_csr(golden, "c1/ML")))
    # spmm (dense.hpp:41) through the block kernel: bitwise the per-column spmv
    # and the oracle's spmv of every column
    assert bitwise_equal(dump["spmm11"], dump["spmm11_cols"])
    n = golden_csr(golden, "c1/ML").nrows
    want = np.concatenate([port.spmv(golden_csr(golden, "c1/ML"), O.uniform_pm1(40 + j, n)) for j in range(11)])
    assert bitwise_equal(dump["spmm11"], want)
    r = golden["c1/r"]
    assert bitwise_equal(dump["sweeps"], port.jacobi_sweeps_apply(L, True, r, 4))
    _, tt = port.jacobi_split(U, False)
    from oracle.oracle import Csr  # noqa: F401

    A = golden_csr(golden, "c1/A")
    assert dump["ilu_res"][0] <= 1e-12 * 8
    ML, MU = golden_csr(golden, "c1/ML"), golden_csr(golden, "c1/MU")
    xo, so = O.gmres(A, ML, MU, r, 30, 1e-8, 3000)
    assert dump["gmres_iters"][0] == so["iterations"]
    assert bitwise_equal(dump["gmres_x"], xo) and bitwise_equal(dump["gmres_hist"], so["history"])


def test_shim_device_ilu_path_identical(dump, tmp_path):
    """The shim's ilu_k takes the device factorization for large matrices;
    forcing it for every size (SAIT_SHIM_DEVICE_ILU_MIN=0) changes no output."""
    exe = os.path.join(ROOT, "build", "shim_check")
    path = str(tmp_path / "out_dev.bin")
    env = dict(os.environ, SAIT_SHIM_DEVICE_ILU_MIN="0")
    r = subprocess.run([exe, path], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    dev = read_dump(path)
    assert dev.keys() == dump.keys()
    for k in dump:
        assert np.array_equal(dev[k].view(np.uint8), dump[k].view(np.uint8)), k


def test_shim_exceptions(dump):
    msg = lambda k: bytes(dump[k].astype(np.uint8)).decode()  # noqa: E731
    assert msg("err_thr") == "sait_thr: threshold must be in [0, 1), got 1.500000"
    assert msg("err_diag") == "jacobi_split: singular matrix, zero diagonal at row 5"
    assert msg("err_apply") == "spmv: vector length 5 does not match ncols 4096"
    assert msg("err_trisolve") == "trisolve: singular matrix, zero diagonal at row 9"
    assert msg("err_droprule").startswith("sait_polynomial: a custom DropRule cannot run on the device")
