"""GPU parity of the SAIT apply z = M_U (M_L r) and the block apply against the
reference's own outputs (golden) and the oracle port: bitwise, since each row
is summed sequentially in stored order without FMA (kernels.cpp:18-24)."""
import numpy as np
import pytest

from conftest import golden_csr
from helpers import bitwise_equal, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


@pytest.fixture(scope="module")
def c1_pair(S, golden):
    ML = to_product(golden_csr(golden, "c1/ML"))
    MU = to_product(golden_csr(golden, "c1/MU"))
    return S.SaitPairPreconditioner(ML, MU)


def test_c1_apply_host(S, golden, c1_pair):
    z = np.empty(4096)
    c1_pair.apply(golden["c1/r"], z)
    assert bitwise_equal(z, golden["c1/z"])
    assert c1_pair.name() == "sait" and c1_pair.nnz() == 2 * 51215


def test_c1_apply_device(S, golden, c1_pair):
    import torch

    r = torch.from_numpy(golden["c1/r"]).cuda()
    z = torch.empty_like(r)
    c1_pair.apply(r, z)
    torch.cuda.synchronize()
    assert bitwise_equal(z.cpu().numpy(), golden["c1/z"])


def test_c1_apply_block(S, golden, c1_pair):
    import torch

    Z = c1_pair.apply_block(golden["c1/R8"])
    assert bitwise_equal(np.asfortranarray(Z).ravel(order="F"), np.asfortranarray(golden["c1/Z8"]).ravel(order="F"))
    # device, row-major layout
    R = torch.from_numpy(np.ascontiguousarray(golden["c1/R8"])).cuda()
    Zd = c1_pair.apply_block(R, layout="row")
    torch.cuda.synchronize()
    assert bitwise_equal(Zd.cpu().numpy(), golden["c1/Z8"])


@pytest.mark.parametrize("nvec", [1, 2, 3, 5, 8, 11, 16])
def test_block_widths(S, golden, c1_pair, nvec):
    from oracle import oracle as O

    R = np.stack([O.uniform_pm1(900 + c, 4096) for c in range(nvec)], axis=1)
    Z = c1_pair.apply_block(R)
    for c in range(nvec):
        z = np.empty(4096)
        c1_pair.apply(np.ascontiguousarray(R[:, c]), z)
        assert bitwise_equal(Z[:, c], z)


def test_block_host_pipeline_pinned(S, c1_pair, monkeypatch):
    """apply_block on host vectors pipelines H2D / pair / D2H per vector over
    three device slots; pinned caller buffers, z passed in, more vectors than
    slots: bitwise equal to the unpipelined block path and to single applies."""
    import torch
    from oracle import oracle as O

    nvec = 10
    Rh = torch.empty((nvec, 4096), dtype=torch.float64).pin_memory()
    Zh = torch.zeros((nvec, 4096), dtype=torch.float64).pin_memory()
    for c in range(nvec):
        Rh[c].copy_(torch.from_numpy(O.uniform_pm1(700 + c, 4096)))
    Rn, Zn = Rh.numpy(), Zh.numpy()
    assert c1_pair.apply_block(Rn.T, Zn.T) is not None
    monkeypatch.setenv("SAIT_BLOCK_HOST_PIPELINE", "0")
    Z0 = c1_pair.apply_block(Rn.T)
    assert bitwise_equal(Zn.T, Z0)
    for c in range(nvec):
        z = np.empty(4096)
        c1_pair.apply(Rn[c], z)
        assert bitwise_equal(Zn[c], z)
    with pytest.raises(TypeError):
        c1_pair.apply_block(Rn.T, Zn)  # C-ordered (nvec, n): wrong shape / order


@pytest.mark.parametrize("pin_r,pin_z", [(False, False), (False, True), (True, False)])
def test_block_host_pipeline_pageable_staging(S, c1_pair, monkeypatch, pin_r, pin_z):
    """apply_block on PAGEABLE caller blocks (the reference's std::vector
    callers, preconditioner.cpp:47-49): r and/or z pass through the library's
    pinned staging slots, copied by the host cores.  More groups than slots and
    a ragged last group; every pinned/pageable combination; with one and with
    several copying threads; bitwise the unstaged block path and the single
    applies.  A second call reuses the slots."""
    import torch
    from oracle import oracle as O

    nvec = 19
    R = np.asfortranarray(np.stack([O.uniform_pm1(900 + c, 4096) for c in range(nvec)], axis=1))
    Rt = torch.from_numpy(R.T.copy())  # (nvec, n) C-order = column-major (n, nvec)
    Zt = torch.zeros_like(Rt)
    if pin_r:
        Rt = Rt.pin_memory()
    if pin_z:
        Zt = Zt.pin_memory()
    Rn, Zn = Rt.numpy(), Zt.numpy()
    for _ in range(2):
        Zn[...] = 0.0
        assert c1_pair.apply_block(Rn.T, Zn.T) is not None
        for c in range(nvec):
            z = np.empty(4096)
            c1_pair.apply(np.ascontiguousarray(Rn[c]), z)
            assert bitwise_equal(Zn[c], z)
    monkeypatch.setenv("SAIT_BLOCK_HOST_PIPELINE", "0")
    Z0 = c1_pair.apply_block(Rn.T)
    assert bitwise_equal(Zn.T, Z0)


def test_block_host_pageable_staging_parallel_copies(S, monkeypatch):
    """the staged pageable block apply at a size whose groups are copied by
    several host threads (n = 64^3: 8 MB groups, 1 MB pieces); bitwise the
    device block apply"""
    import torch

    A = S.laplacian_3d(64)
    f = S.ilu_k(A, 0)
    ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
    pair = S.SaitPairPreconditioner(ML, MU)
    nvec, n = 15, A.nrows
    Rn = np.stack([S.uniform_pm1(40 + c, n) for c in range(nvec)])  # (nvec, n), pageable
    Zn = np.zeros_like(Rn)
    pair.apply_block(Rn.T, Zn.T)
    Zd = torch.empty((nvec, n), dtype=torch.float64, device="cuda")
    pair.apply_block(torch.from_numpy(Rn).cuda().T, Zd.T)
    torch.cuda.synchronize()
    assert bitwise_equal(Zn, Zd.cpu().numpy())


def test_host_paths_share_stream_work(S):
    """the block pipeline, the chunked single-vector host apply and the device
    apply share one per-stream workspace: any order of calls on one thread
    works (n >= 2^17 so the single-vector host apply takes the chunked path)"""
    import torch
    from oracle import oracle as O

    A = S.laplacian_3d(52)
    f = S.ilu_device(A, 0)
    pair = S.SaitPairPreconditioner(S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3)),
                                    S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3)))
    n = A.nrows
    R = np.stack([O.uniform_pm1(40 + c, n) for c in range(4)], axis=1)
    want = []
    for c in range(4):
        zd = torch.empty(n, dtype=torch.float64, device="cuda")
        pair.apply(torch.from_numpy(np.ascontiguousarray(R[:, c])).cuda(), zd)
        torch.cuda.synchronize()
        want.append(zd.cpu().numpy())
    Z = pair.apply_block(R)
    z = np.empty(n)
    pair.apply(np.ascontiguousarray(R[:, 1]), z)
    Z2 = pair.apply_block(R[:, 1:])
    for c in range(4):
        assert bitwise_equal(Z[:, c], want[c])
    assert bitwise_equal(z, want[1])
    for c in range(3):
        assert bitwise_equal(Z2[:, c], want[c + 1])


def test_spmv_long_and_empty_rows(S, port):
    """rows longer than the 2048-entry staging chunk, empty rows, n % 256 != 0"""
    import scipy.sparse as sp

    rng = np.random.default_rng(7)
    n = 1000
    dense_rows = {3: 5000, 500: 2048, 501: 2049, 999: 7000}
    rows, cols = [], []
    for i in range(n):
        k = dense_rows.get(i, int(rng.integers(0, 9)))
        c = np.sort(rng.choice(8000, size=k, replace=False))
        rows += [i] * k
        cols += list(c)
    vals = rng.standard_normal(len(rows))
    a = sp.csr_matrix((vals, (rows, cols)), shape=(n, 8000))
    a.sort_indices()
    A = S.CsrMatrix.from_scipy(a)
    x = rng.standard_normal(8000)
    y = S.spmv(A, x)
    from helpers import to_oracle

    assert bitwise_equal(y, port.spmv(to_oracle(A), x))


def test_apply_errors(S, c1_pair):
    with pytest.raises(S.SaitInvalidArgument, match="spmv: vector length 5 does not match ncols 4096"):
        c1_pair.apply(np.zeros(5), np.zeros(4096))
    with pytest.raises(S.SaitInvalidArgument, match="spmv: output length mismatch"):
        c1_pair.apply(np.zeros(4096), np.zeros(7))
    a = S.CsrMatrix(3, 4, [0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])
    b = S.CsrMatrix(3, 3, [0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])
    with pytest.raises(S.SaitInvalidArgument, match="SaitPairPreconditioner: factor shapes do not chain"):
        S.SaitPairPreconditioner(b, a)


def _pair_from_scipy(S, lo, up):
    return S.SaitPairPreconditioner(S.CsrMatrix.from_scipy(lo), S.CsrMatrix.from_scipy(up))


def test_irregular_pair_falls_back_and_matches(S, port):
    """A pair whose rows are too irregular for the SELL-32 copy (a few very
    long rows) takes the CSR kernels; results stay bitwise equal."""
    import scipy.sparse as sp

    from helpers import to_oracle

    rng = np.random.default_rng(3)
    n = 3000
    lo = sp.tril(sp.random(n, n, density=0.002, random_state=4), k=-1).tolil()
    for i in (100, 2000, 2999):
        lo[i, : i] = rng.standard_normal(i)
    lo = (lo + sp.eye(n)).tocsr()
    up = lo.T.tocsr()
    pair = _pair_from_scipy(S, lo, up)
    r = rng.standard_normal(n)
    z = np.empty(n)
    pair.apply(r, z)
    L, U = S.CsrMatrix.from_scipy(lo), S.CsrMatrix.from_scipy(up)
    assert bitwise_equal(z, port.pair_apply(to_oracle(L), to_oracle(U), r))
    Z = pair.apply_block(np.stack([r, -r, 2 * r, r], axis=1))
    assert bitwise_equal(Z[:, 0], z)


def test_nonfinite_inputs_propagate_like_reference(S, golden, c1_pair, port):
    """Padding slots of the sliced format are never multiplied: an Inf/NaN in
    r reaches exactly the rows the reference reaches."""
    from helpers import to_oracle

    r = golden["c1/r"].copy()
    r[17] = np.inf
    r[2048] = np.nan
    z = np.empty(4096)
    c1_pair.apply(r, z)
    ML = to_product(golden_csr(golden, "c1/ML"))
    MU = to_product(golden_csr(golden, "c1/MU"))
    ez = port.pair_apply(to_oracle(ML), to_oracle(MU), r)
    assert np.array_equal(np.isnan(z), np.isnan(ez)) and np.array_equal(np.isinf(z), np.isinf(ez))
    fin = np.isfinite(ez)
    assert bitwise_equal(z[fin], ez[fin])


@pytest.mark.parametrize("sched,zc", [("default", "1"), ("0.5;0.5;0.25", "1"), ("0.5;0.5;0.25", "0"),
                                       ("0.25,0.5;0.75;0.5,0.25", "1"), ("0.5,0.5,0.25", "0")])
def test_chunked_host_apply_3d(S, port, sched, zc, monkeypatch):
    """Host-vector apply on n = 64^3 through the chunked PCIe pipeline (chunk
    schedules small enough for several chunks; z by zero-copy stores or by
    copy-engine D2H): bitwise equal to the device-vector apply and the oracle."""
    import torch

    from helpers import to_oracle

    if sched != "default":
        monkeypatch.setenv("SAIT_PIPE_MB", sched)
    monkeypatch.setenv("SAIT_HOST_ZC_OUT", zc)

    A = S.laplacian_3d(64)
    f = S.ilu_k(A, 0)
    ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
    pair = S.SaitPairPreconditioner(ML, MU)
    ez = port.pair_apply(to_oracle(ML), to_oracle(MU), S.uniform_pm1(7, A.nrows))
    for pinned in (False, True):
        r = torch.from_numpy(S.uniform_pm1(7, A.nrows))
        z = torch.empty_like(r)
        if pinned:
            r, z = r.pin_memory(), z.pin_memory()
        for _ in range(2):  # second call reuses the cached pipeline
            z.zero_()
            pair.apply(r.numpy(), z.numpy())
            assert bitwise_equal(z.numpy(), ez)
    rd = torch.from_numpy(S.uniform_pm1(7, A.nrows)).cuda()
    zd = torch.empty_like(rd)
    pair.apply(rd, zd)
    torch.cuda.synchronize()
    assert bitwise_equal(zd.cpu().numpy(), ez)


FORMATS = ["auto", "csr", "sell32_int32", "sell32_int16", "sell32_dict"]


@pytest.mark.parametrize("fmt", FORMATS)
def test_forced_apply_formats(S, port, fmt):
    """sait_pair_create_ex: every apply storage (CSR, SELL-32 with int32
    columns / int16 deltas / shared slice patterns) gives the oracle's bits
    for the single apply, the block apply and the host apply, and
    sait_pair_format reports the storage and its stream bytes."""
    import torch

    from helpers import to_oracle

    A = S.laplacian_3d(24)
    f = S.ilu_k(A, 0)
    ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
    eL, eU = to_oracle(ML), to_oracle(MU)
    pair = S.SaitPairPreconditioner(ML, MU, format=fmt)
    n = A.nrows
    for w in (0, 1):
        info = pair.factor_format(w)
        want = "sell32_dict" if fmt == "auto" else fmt
        assert info["format"] == want
        nnz = (ML if w == 0 else MU).nnz()
        assert info["nnz"] == nnz and info["stored_slots"] >= nnz
        per = {"csr": 12, "sell32_int32": 12, "sell32_int16": 10, "sell32_dict": 8}[want]
        assert info["stream_bytes"] >= per * info["stored_slots"] + 16 * n
    r = S.uniform_pm1(11, n)
    z = np.empty(n)
    pair.apply(r, z)
    assert bitwise_equal(z, port.pair_apply(eL, eU, r))
    rd = torch.from_numpy(r).cuda()
    zd = torch.empty_like(rd)
    pair.apply(rd, zd)
    torch.cuda.synchronize()
    assert bitwise_equal(zd.cpu().numpy(), z)
    R = np.stack([S.uniform_pm1(20 + j, n) for j in range(8)], axis=1)
    Z = pair.apply_block(R)
    assert bitwise_equal(np.asarray(Z), port.pair_apply_block(eL, eU, R))
    with pytest.raises(ValueError):
        S.SaitPairPreconditioner(ML, MU, format="ellpack")


@pytest.mark.parametrize("fmt", ["auto", "sell32_int32", "sell32_int16"])
def test_ragged_factor_row_sorted(S, port, fmt):
    """A factor too ragged for 32-row slices in its natural order (the SAIT
    factor of config 4's T^T: padding > 25%) gets a SELL copy with its rows
    sorted by length within 1024-row windows (SELL-C-sigma, row_sorted); the
    single apply (device and host vectors) and the block apply (column- and
    row-major) keep the oracle's bits."""
    import torch

    from helpers import to_oracle

    T = S.synthetic_lower(1 << 14, 15, 0.01, 4)
    M = S.sait_thr(T, S.lower_triangular, S.SaitThrParams(1e-2, 3))
    Mt = S.transpose(M)
    pair = S.SaitPairPreconditioner(M, Mt, format=fmt)
    fu = pair.factor_format(1)
    assert fu["row_sorted"] and fu["format"] == ("sell32_int32" if fmt == "sell32_int32" else "sell32_int16")
    assert fu["stored_slots"] <= 1.25 * fu["nnz"] + 64
    eL, eU = to_oracle(M), to_oracle(Mt)
    n = M.nrows
    r = S.uniform_pm1(5, n)
    want = port.pair_apply(eL, eU, r)
    z = np.empty(n)
    pair.apply(r, z)
    assert bitwise_equal(z, want)
    rd = torch.from_numpy(r).cuda()
    zd = torch.empty_like(rd)
    pair.apply(rd, zd)
    torch.cuda.synchronize()
    assert bitwise_equal(zd.cpu().numpy(), want)
    R = np.stack([S.uniform_pm1(40 + j, n) for j in range(8)], axis=1)
    Zb = port.pair_apply_block(eL, eU, R)
    assert bitwise_equal(np.asarray(pair.apply_block(R)), Zb)
    Rd = torch.from_numpy(np.ascontiguousarray(R.T)).cuda()  # (8, n): the column-major (n, 8) block
    Zd = torch.empty_like(Rd)
    pair.apply_block(Rd.T, Zd.T)
    torch.cuda.synchronize()
    assert bitwise_equal(Zd.T.cpu().numpy(), Zb)
    Rr = torch.from_numpy(np.ascontiguousarray(R)).cuda()  # (n, 8) row-major
    Zr = pair.apply_block(Rr, layout="row")
    torch.cuda.synchronize()
    assert bitwise_equal(Zr.cpu().numpy(), Zb)


_DICT_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import ctypes as C
import paper_2106_12836_b200 as S
from paper_2106_12836_b200 import _native as N
from oracle import oracle as O
P = O.get("port")
A = O.laplacian_3d(24)
L, U = P.ilu_k(A, 0)
ML, MU = P.sait_thr(L, True, 5e-2, 3), P.sait_thr(U, False, 5e-2, 3)
from helpers import to_product
pair = S.SaitPairPreconditioner(to_product(ML), to_product(MU))
N.lib.sait_debug_pair_index_kind.restype = C.c_int
kinds = [N.lib.sait_debug_pair_index_kind(pair.handle, w) for w in (0, 1)]
r = O.uniform_pm1(3, A.nrows)
z = np.empty(A.nrows)
pair.apply(r, z)
ok = np.array_equal(z.view(np.uint64), P.pair_apply(ML, MU, r).view(np.uint64))
print(kinds[0], kinds[1], int(ok))
"""


@pytest.mark.parametrize("env,index,kind", [("1", "", 2), ("0", "", 1), ("1", "32", 2), ("0", "32", 0)])
def test_sell_index_formats(env, index, kind):
    """The SELL copy of a stencil factor uses shared slice patterns (a few
    distinct delta blocks serve every slice, built from int16 deltas or from
    int32 columns) unless SAIT_SELL_DICT=0; every format gives the oracle's
    bits."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    code = _DICT_CHILD.format(root=ROOT)
    envd = dict(os.environ, SAIT_SELL_DICT=env, PYTHONPATH=os.path.join(ROOT, "tests"))
    if index:
        envd["SAIT_SELL_INDEX"] = index
    out = subprocess.run([sys.executable, "-c", code], env=envd, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    k0, k1, ok = map(int, out.stdout.split()[-3:])
    assert (k0, k1, ok) == (kind, kind, 1)


@pytest.mark.parametrize("sched", ["0.5;0.5;0.25", "default"])
def test_concurrent_applies_from_threads(S, port, sched, monkeypatch):
    """apply is const and safe to call concurrently (preconditioner.hpp:15-16):
    host-vector applies from 4 threads (each gets its own internal stream),
    device applies from 4 threads of which two share torch's default stream
    (their launches take turns) and two have their own streams."""
    import threading

    import torch

    from helpers import to_oracle

    if sched != "default":
        monkeypatch.setenv("SAIT_PIPE_MB", sched)
    A = S.laplacian_3d(64)
    f = S.ilu_k(A, 0)
    ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
    pair = S.SaitPairPreconditioner(ML, MU)
    n = A.nrows
    rs = [S.uniform_pm1(300 + i, n) for i in range(8)]
    want = [port.pair_apply(to_oracle(ML), to_oracle(MU), r) for r in rs]
    errors = []

    def host_worker(i):
        try:
            r = torch.from_numpy(rs[i]).pin_memory() if i % 2 else torch.from_numpy(rs[i])
            z = torch.empty(n, dtype=torch.float64)
            z = z.pin_memory() if i % 2 else z
            for _ in range(5):
                z.zero_()
                pair.apply(r.numpy(), z.numpy())
                if not bitwise_equal(z.numpy(), want[i]):
                    errors.append(("host", i))
        except Exception as e:  # noqa: BLE001
            errors.append(("host", i, repr(e)))

    def dev_worker(i, own_stream):
        try:
            st = torch.cuda.Stream() if own_stream else torch.cuda.default_stream()
            with torch.cuda.stream(st):
                r = torch.from_numpy(rs[i]).cuda()
                z = torch.empty_like(r)
                for _ in range(5):
                    pair.apply(r, z)
                st.synchronize()
                if not bitwise_equal(z.cpu().numpy(), want[i]):
                    errors.append(("dev", i))
        except Exception as e:  # noqa: BLE001
            errors.append(("dev", i, repr(e)))

    th = [threading.Thread(target=host_worker, args=(i,)) for i in range(4)]
    th += [threading.Thread(target=dev_worker, args=(4 + i, i >= 2)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
