#!/usr/bin/env python3
"""bench.py — BASELINE.json's headline metric on B200.

Workload (BASELINE.json configs[1], "config 2"): 3D 7-point Laplacian 128^3
(n = 2,097,152), ILU(0), SAIT tau = 5e-2, k = 3 for both factors; one STEP =
the SAIT apply z = M_U (M_L r) on 100 seeded U[-1,1] vectors (seeds
1000..1099), applied one after the other (one SpMV pair each).

  value      algorithmic GB/s of the pair, inputs resident in HBM:
             100 * B_pair / t_step,  B_pair = 12 (nnz_L + nnz_U) + 8 (n+1) + 32 n
  e2e        the same metric through the public host-vector API: the step's
             100 vectors as one apply_block call on the pinned (n, 100) host
             block (sait_pair_apply_block_host: H2D, pairs, D2H pipelined per
             group of vectors); the per-vector apply loop is reported beside it
  roofline   dominant kernel (the SpMV) achieved GB/s vs MEASURED_PEAKS.json
  cpu_baseline  the reference (oracle/_ref, compiled from the reference's own
             sources) timed on this host, all threads, bounded sample
  build      SAIT build of both factors on device: built nnz/s

`--impl reference` times the reference's own CPU path (SaitPairPreconditioner::
apply from oracle/_ref) on the same workload and prints the same JSON line.
Inputs larger than L2: the two factors stream 349 MB per pair (> 126 MB L2),
so no explicit flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# rank 0 prints exactly one JSON line on stdout: keep NCCL's version banner
# (NCCL_DEBUG=VERSION prints it to stdout) off it
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"

BASE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASE["metric"]
BUILD_REPS = 5
GRID = 128
TAU, STEPS_K = 5e-2, 3
NVEC = 100
SEED0 = 1000
WORKLOAD = "c2: laplacian3d 128^3, ILU(0), SAIT_thr(tau=5e-2, k=3), apply pair x100 vectors"


def b_pair(n, nnz_l, nnz_u):
    return 12 * (nnz_l + nnz_u) + 8 * (n + 1) + 32 * n


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.out = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.out.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


def bench_config(n, nnz_l, nnz_u, ws):
    """The workload keys both arms print (same_config)."""
    return {"workload": WORKLOAD, "n": n, "nnz_L": nnz_l, "nnz_U": nnz_u, "bytes_per_pair": b_pair(n, nnz_l, nnz_u),
            "vectors_per_step": NVEC, "parallelism": f"rows{ws}" if ws > 1 else "single",
            "l2": "inputs larger than L2: 349 MB of factors streamed per pair (> 126 MB L2), no flush"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------- reference arm

def ref_inputs(O, R):
    A = O.laplacian_3d(GRID)
    L, U = R.ilu_k(A, 0)
    return A, L, U


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone times the CPU reference
    from oracle import oracle as O

    if not O.ref_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libsaitref.so not built"})
        return
    import ctypes as C

    R = O.get("reference")
    A, L, U = ref_inputs(O, R)
    tb0 = time.perf_counter()
    ML = R.sait_thr(L, True, TAU, STEPS_K)
    MU = R.sait_thr(U, False, TAU, STEPS_K)
    t_build = time.perf_counter() - tb0
    n = A.nrows
    B = b_pair(n, ML.nnz, MU.nnz)
    lib = R.lib
    lib.ref_pair_create.restype = C.c_void_p
    lib.ref_pair_create.argtypes = [C.c_void_p, C.c_void_p]
    lib.ref_pair_time_apply.restype = C.c_double
    lib.ref_pair_time_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64]
    from oracle.oracle import _in

    p = lib.ref_pair_create(C.byref(_in(ML)), C.byref(_in(MU)))
    sample = int(os.environ.get("SAIT_REF_SAMPLE", "20"))  # vectors per step (bounded sample)
    r = np.stack([O.uniform_pm1(SEED0 + i, n) for i in range(sample)])
    z = np.empty_like(r)
    for _ in range(args.warmup):
        lib.ref_pair_time_apply(p, r.ctypes.data, z.ctypes.data, n, sample)
    ts = [lib.ref_pair_time_apply(p, r.ctypes.data, z.ctypes.data, n, sample) for _ in range(args.steps)]
    t = float(np.sum(ts))
    value = sample * args.steps * B / t / 1e9
    cores = int(lib.ref_max_threads())
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps * NVEC / sample,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(n, ML.nnz, MU.nnz, ws),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": f"{sample} vectors per step through SaitPairPreconditioner::apply (OpenMP {cores} threads)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build": {"built_nnz": ML.nnz + MU.nnz, "seconds": t_build, "nnz_per_s": (ML.nnz + MU.nnz) / t_build,
                  "note": f"the reference's sait_thr on L then U (OpenMP {cores} threads), one build each"},
    }
    if not args.no_c4:
        line["build_c4"] = c4_reference_sample()
    lib.ref_pair_destroy.argtypes = [C.c_void_p]
    lib.ref_pair_destroy(p)
    emit(line)


# --------------------------------------------------------------------- B200 arm

def cpu_baseline_sample(ML_host, MU_host, n):
    """The reference's apply on the GPU-built factors (bitwise identical to the
    reference's own), timed on this host's cores.  Returns dict or None."""
    from oracle import oracle as O

    if not O.ref_available():
        return None
    import ctypes as C

    from oracle.oracle import Csr, _in

    R = O.get("reference")
    lib = R.lib
    lib.ref_pair_create.restype = C.c_void_p
    lib.ref_pair_create.argtypes = [C.c_void_p, C.c_void_p]
    lib.ref_pair_time_apply.restype = C.c_double
    lib.ref_pair_time_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64]
    ml = Csr(ML_host.nrows, ML_host.ncols, ML_host.row_ptr, ML_host.col_idx, ML_host.values)
    mu = Csr(MU_host.nrows, MU_host.ncols, MU_host.row_ptr, MU_host.col_idx, MU_host.values)
    p = lib.ref_pair_create(C.byref(_in(ml)), C.byref(_in(mu)))
    # bounded sample: whole 100-vector steps until ~10 s of CPU work (max 30 steps)
    budget = float(os.environ.get("SAIT_CPU_SECONDS", "10"))
    r = np.stack([O.uniform_pm1(SEED0 + i, n) for i in range(NVEC)])
    z = np.empty_like(r)
    lib.ref_pair_time_apply(p, r.ctypes.data, z.ctypes.data, n, 2)  # warm
    t, steps = 0.0, 0
    while t < budget and steps < 30:
        t += lib.ref_pair_time_apply(p, r.ctypes.data, z.ctypes.data, n, NVEC)
        steps += 1
    B = b_pair(n, ml.nnz, mu.nnz)
    cores = int(lib.ref_max_threads())
    # SURVEY.md §8(d) timing protocol extras (bounded): y preallocated (all
    # threads, the reference's per-call allocation removed) and 1 thread
    extra = {}
    try:
        lib.ref_pair_time_apply_prealloc.restype = C.c_double
        lib.ref_pair_time_apply_prealloc.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64]
        tp = lib.ref_pair_time_apply_prealloc(p, r.ctypes.data, z.ctypes.data, n, NVEC)
        extra["prealloc_y"] = {"value": NVEC * B / tp / 1e9, "cores": cores, "sample": f"{NVEC} vectors, {tp:.2f} s"}
        lib.ref_set_threads.argtypes = [C.c_int]
        lib.ref_set_threads(1)
        n1 = 10
        t1 = lib.ref_pair_time_apply(p, r.ctypes.data, z.ctypes.data, n, n1)
        lib.ref_set_threads(cores)
        extra["single_thread"] = {"value": n1 * B / t1 / 1e9, "cores": 1, "sample": f"{n1} vectors, {t1:.2f} s"}
    except AttributeError:
        pass
    lib.ref_pair_destroy.argtypes = [C.c_void_p]
    lib.ref_pair_destroy(p)
    return {"value": steps * NVEC * B / t / 1e9, "unit": "GB/s", "cores": cores, "kind": "reference",
            "sample": f"{steps} steps x 100 vectors through the reference SaitPairPreconditioner::apply "
                      f"(oracle/_ref, OpenMP {cores} threads), {t:.1f} s",
            "ms_per_step": 1e3 * t / steps, **extra}


def time_steps(step, steps, stream, torch):
    """ms per step of `step()` (one warm-up step, CUDA events on `stream`)."""
    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def apply_format_lines(S, torch, Ld, Ud, R, Z_ref, steps, stream):
    """The same C2 step with the factors forced into the other apply formats
    (sait_pair_create_ex): int16 column deltas (10 B/nnz), int32 columns
    (12 B/nnz) and plain CSR (the irregular-matrix kernel).  Each line is
    checked bitwise against the default format's outputs."""
    peak, _ = peaks()
    out = {}
    nvec, n = R.shape
    Zv = torch.empty_like(R)
    for fmt in ("sell32_int16", "sell32_int32", "csr"):
        ML, MU = S.sait_thr_pair(Ld, Ud, S.SaitThrParams(TAU, STEPS_K))
        B = b_pair(n, ML.nnz(), MU.nnz())
        pair = S.SaitPairPreconditioner(ML, MU, format=fmt)

        def step():
            for i in range(nvec):
                pair.apply(R[i], Zv[i])

        ms = time_steps(step, steps, stream, torch)
        fl, fu = pair.factor_format(0), pair.factor_format(1)
        fb = fl["stream_bytes"] + fu["stream_bytes"]
        ach = nvec * fb / (ms * 1e-3) / 1e9
        out[fmt] = {"formats": [fl["format"], fu["format"]], "ms_per_step": ms,
                    "effective_gbs_12B_per_nnz": nvec * B / (ms * 1e-3) / 1e9,
                    "format_bytes_per_pair": fb, "achieved": ach, "frac": ach / peak,
                    "bitwise_equal_default_format": bool(torch.equal(Zv, Z_ref))}
        del pair
    return out


def irregular_apply_line(S, torch, T, steps, stream, nvec=20):
    """An apply on an irregular (non-stencil) pattern: the SAIT pair of the
    config-4 generator's T (lower, n = 2^24) and T^T (upper), tau = 1e-2,
    k = 3 -- random geometric column offsets, so no slice patterns repeat, and
    M_U's rows are too ragged for 32-row slices in their natural order: its
    SELL copy sorts them by length within 1024-row windows (SELL-C-sigma)."""
    peak, _ = peaks()
    Tt = S.transpose(T)
    P = S.SaitThrParams(1e-2, 3)
    ML = S.sait_thr(T, S.lower_triangular, P)
    MU = S.sait_thr(Tt, S.upper_triangular, P)
    Tt.free()
    n = T.nrows
    B = b_pair(n, ML.nnz(), MU.nnz())
    nnz = (ML.nnz(), MU.nnz())
    pair = S.SaitPairPreconditioner(ML, MU)
    R = torch.empty((nvec, n), dtype=torch.float64, device="cuda")
    for i in range(nvec):
        R[i].copy_(torch.from_numpy(S.uniform_pm1(SEED0 + i, n)))
    Z = torch.empty_like(R)

    def step():
        for i in range(nvec):
            pair.apply(R[i], Z[i])

    ms = time_steps(step, steps, stream, torch)
    fl, fu = pair.factor_format(0), pair.factor_format(1)
    fb = fl["stream_bytes"] + fu["stream_bytes"]
    ach = nvec * fb / (ms * 1e-3) / 1e9
    del pair, R, Z
    return {"workload": "SAIT pair of the c4 generator's T and T^T (n=2^24), tau=1e-2, k=3, %d vectors per step" % nvec,
            "n": n, "nnz_L": nnz[0], "nnz_U": nnz[1], "formats": [fl["format"], fu["format"]], "row_sorted": [fl["row_sorted"], fu["row_sorted"]],
            "ms_per_step": ms, "ms_per_pair": ms / nvec, "effective_gbs_12B_per_nnz": nvec * B / (ms * 1e-3) / 1e9,
            "format_bytes_per_pair": fb, "achieved": ach, "frac": ach / peak}


# ------------------------------------------------------- N GPUs (row/column shards)

def _max_over_ranks(dist, torch, v: float) -> float:
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(dist, torch, v: int) -> int:
    t = torch.tensor([v], dtype=torch.int64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def sharded_factors(S, torch, dist, Ld, Ud, spec, rank, ws):
    """Both SAIT factors built COLUMN-sharded (each rank the columns of its
    work-balanced block, the global early stop all-reduced per step: the
    reference's step count and bits) and redistributed on the device to the
    apply's row blocks (K4: NCCL point-to-point of the pieces, device
    assembly).  Returns (row blocks, bounds, seconds max over ranks, per-rank
    build info)."""
    from paper_2106_12836_b200.dist import build_sharded, column_bounds_by_work, redistribute_to_rows, row_bounds

    n = Ld.nrows
    rb = row_bounds(n, ws)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    blocks, info = [], []
    for lower, Td in ((True, Ld), (False, Ud)):
        cb = column_bounds_by_work(Td, ws)
        blk, st, (c0, c1) = build_sharded(Td, lower, spec, rank, ws, transposed=False, bounds=cb)
        info.append({"columns": [c0, c1], "nnz": blk.nnz(), "steps_run": st.steps_run, "products": st.products})
        blocks.append(redistribute_to_rows(blk, cb, rb, rank, ws))
        blk.free()
    torch.cuda.synchronize()
    t = _max_over_ranks(dist, torch, time.perf_counter() - t0)
    return blocks, rb, t, info


def run_sharded_c5(S, torch, dist, rank, ws, steps, nvec=20):
    """BASELINE config 5's apply, row-sharded: 256^3 Laplacian, device ILU(0)
    (replicated: each rank factors the whole matrix, 0.1 s), SAIT tau = 5e-2,
    k = 3 built column-sharded and redistributed, z = M_U (M_L r) through
    PeerShardedPair on `nvec` seeded vectors per step (the block-8 apply of
    LOBPCG is 8 of these per block here)."""
    from paper_2106_12836_b200 import _native as N
    from paper_2106_12836_b200.dist import PeerShardedPair

    A = S.laplacian_3d(256)
    n = A.nrows
    dA = S.DeviceCsr.upload(A)
    f = S.ilu0_device(dA)
    dA.free()
    spec = N.DropSpec(N.SAIT_DROP_THRESHOLD, 5e-2, 3, 0, 0, 0.0)
    (bl, bu), rb, t_build, info = sharded_factors(S, torch, dist, f.lower, f.upper, spec, rank, ws)
    f.lower.free()
    f.upper.free()
    nnz_l = _sum_over_ranks(dist, torch, bl.nnz())
    nnz_u = _sum_over_ranks(dist, torch, bu.nnz())
    sp = PeerShardedPair.distributed_from_row_blocks(bl, bu, rb, rank, ws)
    r0, r1 = sp.own
    R = torch.empty((nvec, r1 - r0), dtype=torch.float64, device="cuda")
    for i in range(nvec):
        R[i].copy_(torch.from_numpy(S.uniform_pm1(5000 + i, n)[r0:r1]))
    Z = torch.empty_like(R)

    def step():
        for i in range(nvec):
            sp.apply(R[i], Z[i])

    step()
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = _max_over_ranks(dist, torch, e0.elapsed_time(e1) / steps)
    B = b_pair(n, nnz_l, nnz_u)
    out = {"workload": "c5: laplacian3d 256^3, ILU(0), SAIT_thr(tau=5e-2, k=3), row-sharded apply pair, "
                       "%d vectors per step" % nvec,
           "n": n, "nnz_L": nnz_l, "nnz_U": nnz_u, "bytes_per_pair": B, "n_gpus": ws, "ms_per_step": ms,
           "ms_per_pair": ms / nvec, "value": nvec * B / (ms * 1e-3) / 1e9, "unit": "GB/s",
           "build_sharded_s": t_build, "build_per_rank_rank0": info, "halo_bytes_per_apply_rank0": sp.halo_bytes,
           "transport": "peer memory halo inside the SpMV (PeerShardedPair)"}
    sp.close()
    return out


def run_sharded_c4(S, torch, dist, rank, ws, reps=3):
    """BASELINE config 4 at N ranks: the fill-capped SAIT build of the n = 2^24
    synthetic T, column-sharded over work-balanced blocks (the global early
    stop all-reduced per step), built nnz/s = total nnz / max-over-ranks wall
    time; per-rank balance reported."""
    from paper_2106_12836_b200 import _native as N
    from paper_2106_12836_b200.dist import build_sharded, column_bounds_by_work

    n = 1 << C4_LOG2N
    Th = S.synthetic_lower(n, 15, 0.01, 4)
    T = S.DeviceCsr.upload(Th)
    del Th
    S.reserve_device_pool(max(8 << 30, (40 << 30) // ws))
    spec = N.DropSpec(N.SAIT_DROP_THRESHOLD_CAP, C4_TAU, C4_K, 0, 0, C4_CAP)
    cb = column_bounds_by_work(T, ws)
    secs, mine = [], None
    for rep in range(1 + reps):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        blk, st, (c0, c1) = build_sharded(T, True, spec, rank, ws, transposed=True, bounds=cb)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        tmax = _max_over_ranks(dist, torch, t)
        if rep:
            secs.append(tmax)
        mine = {"columns": [c0, c1], "nnz": blk.nnz(), "seconds": t, "steps_run": st.steps_run,
                "products": st.products}
        blk.free()
    T.free()
    total = _sum_over_ranks(dist, torch, mine["nnz"])
    per_rank = [None] * ws
    dist.all_gather_object(per_rank, mine)
    tm = sorted(secs)[len(secs) // 2]
    return {"workload": "c4: synthetic lower T n=2^24, SAIT_thr(tau=1e-2, k=3), fill cap 3x, column-sharded",
            "n": n, "n_gpus": ws, "built_nnz": total, "seconds": tm, "nnz_per_s": total / tm,
            "samples_s": [round(x, 5) for x in secs], "column_bounds": cb, "per_rank": per_rank,
            "balance": "column blocks cut on the prefix sums of sait_column_work (predicted products)"}


def run_b200_sharded(args):
    """bench.py --gpus N (N > 1; or --sharded-pipeline at N = 1): C2's apply
    row-sharded over the ranks with peer-memory halos, its factors built
    column-sharded and redistributed on the device; plus config 4's
    column-sharded build and config 5's row-sharded apply."""
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2106_12836_b200 as S
    from paper_2106_12836_b200 import _native as N
    from paper_2106_12836_b200.dist import PeerShardedPair

    A = S.laplacian_3d(GRID)
    n = A.nrows
    dA = S.DeviceCsr.upload(A)
    f = S.ilu0_device(dA)
    dA.free()
    S.reserve_device_pool(4 << 30)
    spec = N.DropSpec(N.SAIT_DROP_THRESHOLD, TAU, STEPS_K, 0, 0, 0.0)
    sharded_factors(S, torch, dist, f.lower, f.upper, spec, rank, ws)  # warm-up (pool, clocks)
    (bl, bu), rb, t_build, binfo = sharded_factors(S, torch, dist, f.lower, f.upper, spec, rank, ws)
    nnz_l = _sum_over_ranks(dist, torch, bl.nnz())
    nnz_u = _sum_over_ranks(dist, torch, bu.nnz())
    B = b_pair(n, nnz_l, nnz_u)
    sp = PeerShardedPair.distributed_from_row_blocks(bl, bu, rb, rank, ws)
    r0, r1 = sp.own
    nloc = r1 - r0
    R = torch.empty((NVEC, nloc), dtype=torch.float64, device="cuda")
    for i in range(NVEC):
        R[i].copy_(torch.from_numpy(S.uniform_pm1(SEED0 + i, n)[r0:r1]))
    Z = torch.empty_like(R)

    def step():
        for i in range(NVEC):
            sp.apply(R[i], Z[i])

    for _ in range(args.warmup):
        step()
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    launches0 = S.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = S.launch_count() - launches0
    dist.barrier()
    ms_step = _max_over_ranks(dist, torch, e0.elapsed_time(e1)) / args.steps
    value = NVEC * B / (ms_step * 1e-3) / 1e9

    # e2e: host vectors in, host vectors out, per vector (pinned buffers)
    Rh = R.cpu().pin_memory()
    Zh = torch.empty_like(Rh).pin_memory()
    rd, zd = torch.empty(nloc, dtype=torch.float64, device="cuda"), torch.empty(nloc, dtype=torch.float64, device="cuda")

    def e2e_one(i):
        rd.copy_(Rh[i], non_blocking=True)
        sp.apply(rd, zd)
        Zh[i].copy_(zd, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    e2e_one(0)
    dist.barrier()
    t0 = time.perf_counter()
    for i in range(NVEC):
        e2e_one(i)
    t_e2e = _max_over_ranks(dist, torch, time.perf_counter() - t0)
    ok = bool(torch.equal(Zh, Z.cpu()))
    e2e = {"value": NVEC * B / t_e2e / 1e9, "unit": "GB/s", "h2d_bytes_per_step": NVEC * 8 * n,
           "d2h_bytes_per_step": NVEC * 8 * n, "ms_per_step": t_e2e * 1e3,
           "api": "per vector: pinned host rows -> device, PeerShardedPair.apply, device -> host (each rank its rows)"}
    halo = sp.halo_bytes
    sp.close()
    c5 = run_sharded_c5(S, torch, dist, rank, ws, max(1, min(args.steps, 3))) if not args.no_c5 else None
    c4 = run_sharded_c4(S, torch, dist, rank, ws) if not args.no_c4 else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(n, nnz_l, nnz_u, ws),
            "roofline": None, "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "e2e_matches_device": ok,
            "build": {"built_nnz": nnz_l + nnz_u, "seconds": t_build, "nnz_per_s": (nnz_l + nnz_u) / t_build,
                      "note": "both factors column-sharded (work-balanced blocks, global early stop all-reduced) "
                              "and redistributed to row blocks on the device (NCCL point-to-point), max over ranks",
                      "rank0": binfo},
        }
        line["config"]["halo_bytes_per_apply_rank0"] = halo
        line["config"]["halo_transport"] = "peer memory inside the SpMV (PeerShardedPair)"
        if c5:
            line["apply_c5"] = c5
        if c4:
            line["build_c4"] = c4
        emit(line)
    dist.destroy_process_group()


def run_b200(args):
    import torch

    ws, rank, local = dist_env()
    if ws > 1 or args.sharded_pipeline:
        return run_b200_sharded(args)
    torch.cuda.set_device(local)
    dist = None
    import paper_2106_12836_b200 as S

    # ---- inputs (host, then device): not timed
    A = S.laplacian_3d(GRID)
    n = A.nrows
    t_ilu_host = time.perf_counter()
    f = S.ilu_k(A, 0)
    t_ilu_host = time.perf_counter() - t_ilu_host
    Ld = S.DeviceCsr.upload(f.lower)
    Ud = S.DeviceCsr.upload(f.upper)
    torch.cuda.synchronize()
    # ---- build (device): both factors at once (sait_build_pair: the two
    # recursions run concurrently), host wall time around the synchronous
    # call; one warm-up build, then the median of BUILD_REPS builds (the GPU
    # clocks ramp during the first build after the host-side setup)
    # the library's device pool grown once up front (sait_device_pool_reserve),
    # as an application that builds repeatedly would do
    S.reserve_device_pool(4 << 30)
    secs, first = [], None
    for rep in range(1 + BUILD_REPS):
        st = []
        if rep:
            ML.free()
            MU.free()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ML, MU = S.sait_thr_pair(Ld, Ud, S.SaitThrParams(TAU, STEPS_K), stats_out=st)
        torch.cuda.synchronize()
        if rep:
            secs.append(time.perf_counter() - t0)
        else:
            first = time.perf_counter() - t0
    nnz_l, nnz_u = ML.nnz(), MU.nnz()
    t_build = sorted(secs)[len(secs) // 2]
    build = {
        "built_nnz": nnz_l + nnz_u,
        "seconds": t_build,
        "nnz_per_s": (nnz_l + nnz_u) / t_build,
        "samples_s": [round(x, 6) for x in secs],
        "first_build_s": round(first, 6),
        "steps_run": [st[0].steps_run, st[1].steps_run],
        "products": st[0].products + st[1].products,
        "note": "both factors built concurrently (sait_build_pair), wall time of the call incl. "
                "split/transposes, median of %d builds after a warm-up" % BUILD_REPS,
    }
    # the same build through the drop-in host API: host int64 CSR in, host
    # int64 CSR out (saitprec::sait_thr's contract, sait.cpp:90-101), both
    # uploads and both downloads inside the timed call
    he = []
    for _ in range(3):
        t0 = time.perf_counter()
        hl, hu = S.sait_thr_pair(f.lower, f.upper, S.SaitThrParams(TAU, STEPS_K))
        he.append(time.perf_counter() - t0)
    build["e2e_host"] = {"seconds": float(np.median(he)), "nnz_per_s": (nnz_l + nnz_u) / float(np.median(he)),
                         "bitwise_equal_device_build": bool(np.array_equal(hl.values.view(np.uint64),
                                                                           ML.to_host().values.view(np.uint64))),
                         "api": "sait_thr_pair on host CsrMatrix (int64 row_ptr/col_idx, fp64) in and out: "
                                "upload + narrowing, build, widening + download; median of 3"}
    del hl, hu
    B = b_pair(n, nnz_l, nnz_u)
    stream = torch.cuda.current_stream()
    ML_host = MU_host = None
    if not args.no_cpu_baseline:
        ML_host, MU_host = ML.to_host(), MU.to_host()
    pair = S.SaitPairPreconditioner(ML, MU)
    r0, r1 = 0, n
    apply_dev = lambda r, z: pair.apply(r, z)  # noqa: E731
    nloc = r1 - r0

    from paper_2106_12836_b200 import _native as NN

    # ---- 100 seeded vectors (this rank's rows) resident in HBM
    R = torch.empty((NVEC, nloc), dtype=torch.float64, device="cuda")
    for i in range(NVEC):
        R[i].copy_(torch.from_numpy(S.uniform_pm1(SEED0 + i, n)[r0:r1]))
    Z = torch.empty_like(R)

    def step():
        for i in range(NVEC):
            apply_dev(R[i], Z[i])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = S.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = S.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    ms_step = ms / args.steps
    value = NVEC * B / (ms_step * 1e-3) / 1e9  # whole-job algorithmic GB/s (the global pair)

    # ---- dominant kernel: the SELL SpMV.  The timed step is nothing but the
    # 200 SpMV launches (M_L, M_U per vector, back to back on `stream`), so
    # its average launch time is ms_step / 200 -- measured on the launching
    # stream inside the timed region, inter-launch gaps included.  `frac` is
    # computed on the bytes the factors' storage format must move
    # (sait_pair_format: values + indices / slice patterns + slice offsets +
    # x + y); the SURVEY §8(d) 12 B/nnz figure is reported separately as the
    # "effective" rate (= value).
    roofline = None
    if ws == 1:
        peak, peak_kind = peaks()
        fl, fu = pair.factor_format(0), pair.factor_format(1)
        fmt_pair = fl["stream_bytes"] + fu["stream_bytes"]
        per_launch_ms = ms_step / (2 * NVEC)
        achieved = NVEC * fmt_pair / (ms_step * 1e-3) / 1e9
        traffic = None
        try:  # one ncu --set full capture of the SpMV under the timed condition
            with open(os.path.join(ROOT, "profiles", "r02_sell_spmv_ncu_full.json")) as fh:
                tr = json.load(fh)
            traffic = tr.get("dram_bytes_per_launch_mean")
        except Exception:
            pass
        # isolated per-launch times (each factor 50x on one vector): context only
        kt = {}
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        for which, nm, src, dst in ((0, "M_L", R[0], y), (1, "M_U", y, Z[0])):
            def one():
                NN.check(NN.lib.sait_pair_spmv_factor(pair.handle, which, src.data_ptr(), dst.data_ptr(),
                                                      stream.cuda_stream))
            one()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(50):
                one()
            a1.record(stream)
            torch.cuda.synchronize()
            kt[nm] = a0.elapsed_time(a1) / 50
        roofline = {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "sell_spmv_kernel (M_L then M_U, programmatic dependent launches)",
            "bytes_model": "format stream bytes per pair (sait_pair_format): stored values + index storage "
                           "(here shared slice patterns: one int32 offset per 32-row slice + the dictionary) + "
                           "int64 slice offsets + x read once + y written once, both factors",
            "format_bytes_per_pair": fmt_pair, "formats": {"M_L": fl, "M_U": fu},
            "per_launch_ms": per_launch_ms,
            "per_launch_source": "ms_per_step / 200 launches, CUDA events on the launching stream (timed region)",
            "effective_gbs_12B_per_nnz": value,
            "effective_note": "SURVEY §8(d) algorithmic bytes (12 B/nnz + vectors) per pair / time = `value`; "
                              "exceeds the copy peak because the format streams ~8 B/nnz",
            "traffic_note": "ncu --set full dram__bytes_read+write per SpMV launch, back-to-back pairs on distinct "
                            "vectors, --cache-control none (profiles/r02_sell_spmv_ncu_full.json; the 8-pair metrics "
                            "capture profiles/r02_apply_traffic.json gives 123 MB)",
            "isolated_per_launch_ms": kt,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, burst copy)",
            "frac_vs_nominal_8000": achieved / 8000.0,
        }

    # ---- e2e: public API with pinned host buffers, H2D + apply + D2H per vector
    Rh = torch.empty((NVEC, nloc), dtype=torch.float64).pin_memory()
    Rh.copy_(R.cpu())
    Zh = torch.empty((NVEC, nloc), dtype=torch.float64).pin_memory()
    Rn, Zn = Rh.numpy(), Zh.numpy()
    e2e_one = lambda i: pair.apply(Rn[i], Zn[i])  # noqa: E731  (sait_pair_apply_host)
    # the whole step as ONE public call: apply_block on the (n, 100)
    # column-major block (preconditioner.cpp:47-49, a per-column spmv loop
    # in the reference), the copies of vector v+1 / v-1 overlapping pair v
    e2e_block = lambda: pair.apply_block(Rn.T, Zn.T)  # noqa: E731  (sait_pair_apply_block_host)
    e2e_one(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(NVEC):
        e2e_one(i)
    t_e2e = time.perf_counter() - t0
    e2e = {"value": NVEC * B / t_e2e / 1e9, "unit": "GB/s", "h2d_bytes_per_step": NVEC * 8 * n,
           "d2h_bytes_per_step": NVEC * 8 * n, "ms_per_step": t_e2e * 1e3,
           "api": "100 x SaitPairPreconditioner::apply (sait_pair_apply_host), synchronous"}
    ok = bool(torch.equal(Zh, Z.cpu()))
    if e2e_block is not None:
        Zh.zero_()
        e2e_block()  # warm: slots, streams, events
        ok = ok and bool(torch.equal(Zh, Z.cpu()))
        Zh.zero_()
        tb = []
        for _ in range(3):
            t0 = time.perf_counter()
            e2e_block()
            tb.append(time.perf_counter() - t0)
        ok = ok and bool(torch.equal(Zh, Z.cpu()))
        t_blk = float(np.median(tb))
        per_vec = e2e
        # the reference's caller holds std::vector (pageable) buffers: the same
        # block call on plain numpy (pageable) memory
        Rp = np.array(Rn)  # (100, n) C order: column-major (n, 100) seen through .T
        Zp = np.zeros_like(Rp)
        pair.apply_block(Rp.T, Zp.T)
        tp = []
        for _ in range(3):
            t0 = time.perf_counter()
            pair.apply_block(Rp.T, Zp.T)
            tp.append(time.perf_counter() - t0)
        ok = ok and bool(np.array_equal(Zp.view(np.uint64), Z.cpu().numpy().view(np.uint64)))
        t_pg = float(np.median(tp))
        e2e = {"value": NVEC * B / t_blk / 1e9, "unit": "GB/s", "h2d_bytes_per_step": NVEC * 8 * n,
               "d2h_bytes_per_step": NVEC * 8 * n, "ms_per_step": t_blk * 1e3,
               "api": "SaitPairPreconditioner::apply_block on the (n, 100) pinned host block "
                      "(sait_pair_apply_block_host), median of 3 calls",
               "per_vector_calls": {"value": per_vec["value"], "ms_per_step": per_vec["ms_per_step"],
                                    "api": "100 x SaitPairPreconditioner::apply, pinned host vectors"},
               "pageable_block": {"value": NVEC * B / t_pg / 1e9, "ms_per_step": t_pg * 1e3,
                                  "api": "the same apply_block call on pageable (plain numpy / std::vector) "
                                         "host memory (groups staged through the library's pinned slots by the host cores), median of 3 calls"}}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(ML_host, MU_host, n)

    # ---- the path's neighbours (not part of `value`): device
    # ILU(0) (F1) against the host factorization, and the exact ILU solves
    # SAIT replaces (F2) against the SAIT apply, same factors, device vectors
    comparators = None
    if ws == 1:
        Ad = S.DeviceCsr.upload(A)
        S.ilu0_device(Ad)  # warm-up (allocator, analysis kernels)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fd = S.ilu0_device(Ad)
        torch.cuda.synchronize()
        t_ilu_dev = time.perf_counter() - t0
        E = S.ExactIluPreconditioner(fd)
        r0v, z0v = R[0], torch.empty_like(R[0])
        E.apply(r0v, z0v)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            E.apply(r0v, z0v)
        torch.cuda.synchronize()
        t_exact = (time.perf_counter() - t0) / 5
        t_sait = ms_step / NVEC * 1e-3
        comparators = {
            "ilu0_device_ms": t_ilu_dev * 1e3, "ilu0_host_ms": t_ilu_host * 1e3,
            "exact_ilu_apply_ms": t_exact * 1e3, "sait_apply_ms": t_sait * 1e3,
            "sait_vs_exact_apply": t_exact / t_sait,
            "note": "F1/F2 (not in value): device ILU(0) bitwise the host ilu_k; exact = two level-scheduled "
                    "device triangular solves, bitwise the reference's trisolve",
        }

    formats = apply_format_lines(S, torch, Ld, Ud, R, Z, max(1, min(args.steps, 3)), stream)
    del R, Z, Rh, Zh
    c5 = None if args.no_c5 else run_c5_single(S, torch, max(1, min(args.steps, 3)), stream)
    solvers = None if args.no_solvers else run_solvers(S, torch, cpu=not args.no_cpu_baseline)

    build_c4 = None
    if not args.no_c4:
        build_c4 = run_build_c4(S, torch, cpu_sample=not args.no_cpu_baseline)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(n, nnz_l, nnz_u, ws),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "build": build, "e2e_matches_device": ok,
        }
        if comparators:
            line["comparators"] = comparators
        if formats:
            line["apply_formats"] = formats
        if c5:
            line["apply_c5"] = c5
        if solvers:
            line["solvers"] = solvers
        if build_c4:
            line["build_c4"] = build_c4
        emit(line)

def run_c5_single(S, torch, steps, stream, nvec=20):
    """BASELINE config 5's preconditioner apply on one GPU: 256^3 Laplacian,
    device ILU(0), SAIT tau = 5e-2, k = 3 (234 M entries): the single-vector
    pair on `nvec` seeded vectors per step, and the block-8 apply (LOBPCG's
    M R, the matrix read once per 8 vectors: apply_block on an (n, 8)
    column-major device block)."""
    peak, _ = peaks()
    A = S.laplacian_3d(256)
    n = A.nrows
    dA = S.DeviceCsr.upload(A)
    f = S.ilu0_device(dA)
    dA.free()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ML, MU = S.sait_thr_pair(f.lower, f.upper, S.SaitThrParams(5e-2, 3))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    nnz_l, nnz_u = ML.nnz(), MU.nnz()
    B = b_pair(n, nnz_l, nnz_u)
    pair = S.SaitPairPreconditioner(ML, MU)
    R = torch.empty((nvec, n), dtype=torch.float64, device="cuda")
    for i in range(nvec):
        R[i].copy_(torch.from_numpy(S.uniform_pm1(5000 + i, n)))
    Z = torch.empty_like(R)

    def step():
        for i in range(nvec):
            pair.apply(R[i], Z[i])

    ms = time_steps(step, steps, stream, torch)
    fl, fu = pair.factor_format(0), pair.factor_format(1)
    fb = fl["stream_bytes"] + fu["stream_bytes"]
    Rb, Zb = R[:8], Z[:8]  # (8, n) row-major = the (n, 8) column-major block

    def blk():
        for _ in range(nvec // 8):
            pair.apply_block(Rb.T, Zb.T)

    ms_b = time_steps(blk, steps, stream, torch) / (nvec // 8)
    B8 = 12 * (nnz_l + nnz_u) + 8 * (n + 1) + 32 * n * 8  # SURVEY §8(d) B_block8
    fb8 = fb + 4 * 8 * 8 * n - 4 * 8 * n  # format bytes with 8 vectors of x/y traffic
    del pair, R, Z
    return {"workload": "c5: laplacian3d 256^3, ILU(0) on device, SAIT_thr(tau=5e-2, k=3), apply pair, "
                        "%d vectors per step; block-8 apply" % nvec,
            "n": n, "nnz_L": nnz_l, "nnz_U": nnz_u, "bytes_per_pair": B, "build_s": t_build,
            "formats": [fl["format"], fu["format"]], "ms_per_pair": ms / nvec,
            "value": nvec * B / (ms * 1e-3) / 1e9, "unit": "GB/s (SURVEY §8(d) algorithmic)",
            "achieved_format_gbs": nvec * fb / (ms * 1e-3) / 1e9, "frac": nvec * fb / (ms * 1e-3) / 1e9 / peak,
            "block8": {"ms": ms_b, "value": B8 / (ms_b * 1e-3) / 1e9, "bytes_block8": B8,
                       "achieved_format_gbs": fb8 / (ms_b * 1e-3) / 1e9, "frac": fb8 / (ms_b * 1e-3) / 1e9 / peak}}


def _host_csr_to_oracle(m):
    from oracle import oracle as O

    return O.Csr(m.nrows, m.ncols, m.row_ptr, m.col_idx, m.values)


def run_solvers(S, torch, cpu=True):
    """The solver loops that drive the apply (north_star (3)), on the device,
    with the restatement (oracle/solvers.c, OpenMP over the host cores, the
    same algorithm and reduction order -- the reference has no solver code,
    SPEC.md:282-351) timed beside them:
      c1  GMRES(30) to 1e-8, 64^2 Poisson, ILU(0), SAIT tau 1e-2 k 4 (full CPU run);
      c3  GMRES(30) to 1e-8, 2048^2 convection-diffusion, tau 2e-2 k 4 (CPU: a
          bounded sample of 60 iterations, per-iteration time reported);
      c5  LOBPCG, 8 pairs, tol 1e-6, 256^3 Laplacian, tau 5e-2 k 3 (CPU:
          the restatement's first 12 iterations recorded when the fixtures
          were made, tests/golden/fullsize.json, not re-run here).
    Each device line carries the preconditioner share of the solve time
    (SolveStats.precond_seconds: the paper's runtime split)."""
    out = {}
    threads = os.cpu_count()
    fix = {}
    try:
        with open(os.path.join(ROOT, "tests", "golden", "fullsize.json")) as fh:
            fix = json.load(fh)
    except Exception:
        pass
    for name, A, tau, k, seed in (("c1", S.laplacian_2d(64), 1e-2, 4, 1),
                                  ("c3", S.convdiff_2d(2048, 20.0, -10.0), 2e-2, 4, 3)):
        dA = S.DeviceCsr.upload(A)
        f = S.ilu0_device(dA)
        ML, MU = S.sait_thr_pair(f.lower, f.upper, S.SaitThrParams(tau, k))
        MLh, MUh = (ML.to_host(), MU.to_host()) if cpu else (None, None)
        pair = S.SaitPairPreconditioner(ML, MU)
        b = S.uniform_pm1(seed, A.nrows)
        bd = torch.from_numpy(b).cuda()
        S.gmres(dA, pair, bd, 30, 1e-8, 20000)  # warm-up (allocations, clocks)
        x, st = S.gmres(dA, pair, bd, 30, 1e-8, 20000)
        line = {"solver": "GMRES(30), right-preconditioned, tol 1e-8", "n": A.nrows, "iterations": st.iterations,
                "converged": st.converged, "true_relres": st.true_relres, "seconds": st.seconds,
                "ms_per_iteration": 1e3 * st.seconds / max(1, st.iterations),
                "precond_seconds": st.precond_seconds, "precond_applies": st.precond_applies,
                "precond_share": st.precond_seconds / st.seconds if st.seconds else None}
        if name == "c3" and "c3" in fix:
            line["restatement_iterations"] = fix["c3"]["gmres"]["iterations"]
        if cpu:
            from oracle import oracle as O

            Ao, Lo, Uo = _host_csr_to_oracle(A), _host_csr_to_oracle(MLh), _host_csr_to_oracle(MUh)
            maxit = 20000 if name == "c1" else 60
            t0 = time.perf_counter()
            _, cs = O.gmres(Ao, Lo, Uo, b, 30, 1e-8, maxit)
            t = time.perf_counter() - t0
            per_it = t / max(1, cs["iterations"])
            line["cpu_baseline"] = {"kind": "port", "cores": threads, "iterations": cs["iterations"],
                                    "seconds": t, "ms_per_iteration": 1e3 * per_it,
                                    "projected_seconds": per_it * st.iterations,
                                    "sample": "full solve" if name == "c1" else
                                    "first 60 iterations (2 restart cycles) of the same solve; projected to the "
                                    "device's iteration count",
                                    "note": "oracle/solvers.c restatement, OpenMP over the host cores (the "
                                            "reference has no GMRES)"}
        out[name] = line
        del pair, x, bd
        dA.free()
    A = S.laplacian_3d(256)
    dA = S.DeviceCsr.upload(A)
    f = S.ilu0_device(dA)
    ML, MU = S.sait_thr_pair(f.lower, f.upper, S.SaitThrParams(5e-2, 3))
    pair = S.SaitPairPreconditioner(ML, MU)
    r = S.lobpcg(dA, pair, 8, 1e-6, 2000, 5, host_vectors=False, gram="tensor")
    rc = S.lobpcg(dA, pair, 8, 1e-6, 2000, 5, host_vectors=False)  # canonical Grams: bitwise the restatement
    st = r.stats
    line = {"solver": "block LOBPCG, 8 smallest pairs, tol 1e-6, SAIT apply_block preconditioner, "
                      "FP64 tensor-core (DMMA) Gram blocks", "n": A.nrows,
            "iterations": r.iterations, "seconds": st.seconds,
            "ms_per_iteration": 1e3 * st.seconds / max(1, r.iterations),
            "max_final_resnorm": float(r.residual_history[-1].max()),
            "precond_seconds": st.precond_seconds, "precond_applies": st.precond_applies,
            "precond_share": st.precond_seconds / st.seconds if st.seconds else None,
            "canonical_grams": {"iterations": rc.iterations, "seconds": rc.stats.seconds,
                                "ms_per_iteration": 1e3 * rc.stats.seconds / max(1, rc.iterations),
                                "note": "the canonical reduction order: bitwise the restatement's run"},
            "max_rel_eig_diff_vs_canonical": float(np.max(np.abs(r.eigenvalues - rc.eigenvalues)
                                                          / np.abs(rc.eigenvalues)))}
    lb = fix.get("c5", {}).get("lobpcg_prefix")
    if lb:
        per_it = lb["cpu_seconds"] / max(1, lb["iterations"])
        line["cpu_baseline"] = {"kind": "port", "cores": lb.get("cpu_threads"), "iterations": lb["iterations"],
                                "seconds": lb["cpu_seconds"], "ms_per_iteration": 1e3 * per_it,
                                "projected_seconds": per_it * rc.iterations,
                                "sample": "the first %d iterations of the same solve, recorded by "
                                          "tests/golden/make_fullsize.py in the build container (not this host), "
                                          "oracle/solvers.c with OpenMP; projected to the device's iteration "
                                          "count" % lb["iterations"]}
    out["c5"] = line
    del pair, r
    dA.free()
    return out


C4_LOG2N, C4_TAU, C4_K, C4_CAP, C4_REPS = 24, 1e-2, 3, 3.0, 3
C4_CPU_LOG2N = 18


def b_build(n, nnz_t, nnz_tt, nnz_steps):
    """SURVEY.md §8(d) algorithmic bytes of one build: the split (T read, tT
    and D^-1 written) plus, per step s, tT + M_{s-1} read, M_s written and
    three int32 row-pointer arrays (M_0 = I)."""
    b = 12 * nnz_t + 12 * nnz_tt + 8 * n
    prev = n
    for m in nnz_steps:
        b += 12 * nnz_tt + 12 * prev + 12 * m + 12 * (n + 1)
        prev = m
    return b


def run_build_c4(S, torch, cpu_sample=True):
    """BASELINE config 4: SAIT build only of the synthetic lower T, n = 2^24
    (15 geometric(0.01) offsets per row, N(0,1) values, d_i = 1.5 sum|t_ij| + 1),
    tau = 1e-2, k = 3, fill cap 3x nnz per column.  Device: median of C4_REPS
    builds after a warm-up (pool reserved up front).  CPU: the reference's own
    sait_thr with the cap through its DropRule hook (oracle/_ref) on a bounded
    n = 2^18 sample of the same generator, checked bitwise against the device
    build of that sample."""
    n = 1 << C4_LOG2N
    t0 = time.perf_counter()
    Th = S.synthetic_lower(n, 15, 0.01, 4)
    t_gen = time.perf_counter() - t0
    T = S.DeviceCsr.upload(Th)
    nnz_t = Th.nnz()
    S.reserve_device_pool(40 << 30)
    P = S.SaitThrParams(C4_TAU, C4_K)
    nnz_steps = []
    for k in range(1, C4_K):  # per-step output sizes for the algorithmic bytes (untimed)
        m = S.sait_thr_cap(T, S.lower_triangular, S.SaitThrParams(C4_TAU, k), C4_CAP)
        nnz_steps.append(m.nnz())
        m.free()
    secs, st = [], []
    for rep in range(1 + C4_REPS):
        st = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = S.sait_thr_cap(T, S.lower_triangular, P, C4_CAP, stats_out=st)
        torch.cuda.synchronize()
        if rep:
            secs.append(time.perf_counter() - t0)
        nnz_m = m.nnz()
        m.free()
    # the drop-in host API end to end: host int64 T in, host int64 M out
    he = []
    for _ in range(2):
        t0 = time.perf_counter()
        Mh = S.sait_thr_cap(Th, S.lower_triangular, P, C4_CAP)
        he.append(time.perf_counter() - t0)
        del Mh
    del Th
    e2e_host = {"seconds": min(he), "nnz_per_s": nnz_m / min(he), "samples_s": [round(x, 4) for x in he],
                "api": "sait_thr_cap on the host CsrMatrix (int64/fp64, 4.2 GB in, 4.4 GB out): upload + narrowing, "
                       "build, widening + download; best of 2"}
    irregular = irregular_apply_line(S, torch, T, 3, torch.cuda.current_stream())
    T.free()
    nnz_steps.append(nnz_m)
    t = sorted(secs)[len(secs) // 2]
    nnz_tt = nnz_t - n
    B = b_build(n, nnz_t, nnz_tt, nnz_steps)
    peak, src = peaks()
    out = {
        "workload": "c4: synthetic lower T n=2^24, SAIT_thr(tau=1e-2, k=3), fill cap 3x nnz(T[:,j])",
        "n": n, "nnz_T": nnz_t, "built_nnz": nnz_m, "nnz_per_step": nnz_steps, "steps_run": st[0].steps_run,
        "products": st[0].products, "seconds": t, "nnz_per_s": nnz_m / t, "samples_s": [round(x, 5) for x in secs],
        "generate_host_s": round(t_gen, 3),
        "roofline": {"bound": "hbm (compulsory bytes; the build is gather/hash-bound)", "algorithmic_bytes": B,
                     "achieved": B / t / 1e9, "peak": peak, "unit": "GB/s", "frac": B / t / 1e9 / peak,
                     "peak_source": src},
        "note": "wall time of the synchronous sait_build call (split, 3 row-form recursion steps, the per-column cap pass after steps 2 and 3), "
                "median of %d after a warm-up" % C4_REPS,
        "irregular_apply": irregular,
        "e2e_host": e2e_host,
    }
    if cpu_sample:
        out["cpu_baseline"] = c4_cpu_sample(S)
    return out


def c4_reference_sample():
    """The reference's capped C4 build on the bounded n = 2^18 sample (no device)."""
    from oracle import oracle as O

    R = O.get("reference")
    T = O.synthetic_lower(1 << C4_CPU_LOG2N, 15, 0.01, 4)
    t0 = time.perf_counter()
    m = R.sait_thr_cap(T, True, C4_TAU, C4_K, C4_CAP)
    t = time.perf_counter() - t0
    return {"value": m.nnz / t, "unit": "built nnz/s", "built_nnz": m.nnz, "seconds": t,
            "sample": f"n=2^{C4_CPU_LOG2N} of the config-4 generator, reference sait_thr + cap DropRule (oracle/_ref)"}


def c4_cpu_sample(S):
    from oracle import oracle as O

    if not O.ref_available():
        return None
    R = O.get("reference")
    n = 1 << C4_CPU_LOG2N
    Th = S.synthetic_lower(n, 15, 0.01, 4)
    To = O.Csr(Th.nrows, Th.ncols, Th.row_ptr, Th.col_idx, Th.values)
    t0 = time.perf_counter()
    ref = R.sait_thr_cap(To, True, C4_TAU, C4_K, C4_CAP)
    t = time.perf_counter() - t0
    dev = S.sait_thr_cap(Th, S.lower_triangular, S.SaitThrParams(C4_TAU, C4_K), C4_CAP)
    same = bool(np.array_equal(dev.row_ptr, ref.row_ptr) and np.array_equal(dev.col_idx, ref.col_idx)
                and np.array_equal(dev.values.view(np.uint64), ref.values.view(np.uint64)))
    import ctypes as C

    lib = R.lib
    lib.ref_max_threads.restype = C.c_int
    return {"value": ref.nnz / t, "unit": "built nnz/s", "cores": int(lib.ref_max_threads()), "kind": "reference",
            "sample": f"n=2^{C4_CPU_LOG2N} of the same generator through the reference sait_thr + cap DropRule "
                      f"(oracle/_ref, OpenMP), {t:.2f} s", "device_bitwise_equal": same}


# The JSON line is the only thing on stdout: libraries that print there
# (NCCL's version banner at communicator creation, CUDA / C printf) write to
# fd 1 directly, so fd 1 is pointed at stderr for the whole run and the line
# goes to the saved original stdout.
_REAL_STDOUT = None


def _claim_stdout():
    global _REAL_STDOUT
    sys.stdout.flush()
    _REAL_STDOUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def emit(line: dict) -> None:
    out = _REAL_STDOUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the BASELINE config-4 build line")
    ap.add_argument("--no-c5", action="store_true", help="skip the BASELINE config-5 apply line")
    ap.add_argument("--no-solvers", action="store_true", help="skip the GMRES (c1, c3) / LOBPCG (c5) lines")
    ap.add_argument("--sharded-pipeline", action="store_true",
                    help="run the N > 1 code path (sharded build, device redistribution, peer-halo apply) at N = 1")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
