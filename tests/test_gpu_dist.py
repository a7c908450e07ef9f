"""Column-block build sessions on the GPU: blocks stepped in lockstep with a
global early-stop reduction must reproduce the single-block build bitwise
(the column form makes every column of M independent).  Plus the row-sharded
pair and the sharded build through torch.distributed (gloo for the host-side
reduction; two processes on one GPU only synchronise on the host)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, golden_csr
from helpers import bitwise_equal, bitwise_equal_csr, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


def _assemble_mt_blocks(blocks, n):
    """Stack M^T row blocks (host CSRs) and transpose to M (host, scipy)."""
    import scipy.sparse as sp

    mt = sp.vstack([b.to_scipy() for b in blocks]).tocsr()
    m = mt.T.tocsr()
    m.sort_indices()
    return m


@pytest.mark.parametrize("kind,args", [("thr", (5e-2, 3)), ("thr", (0.0, 6)), ("pat", (2, 4)), ("cap", (1e-2, 3, 1.5))])
@pytest.mark.parametrize("world", [2, 5])
def test_lockstep_column_blocks_equal_single_build(S, port, kind, args, world):
    from paper_2106_12836_b200 import _native as N
    from paper_2106_12836_b200.dist import row_bounds
    from oracle import oracle as O

    T = O.synthetic_lower(3000, 8, 0.01, seed=13)
    Tp = to_product(T)
    if kind == "thr":
        spec = N.DropSpec(N.SAIT_DROP_THRESHOLD, args[0], args[1], 0, 0, 0.0)
        expect = port.sait_thr(T, True, *args)
    elif kind == "pat":
        spec = N.DropSpec(N.SAIT_DROP_PATTERN, 0.0, 0, args[0], args[1], 0.0)
        expect = port.sait_pat(T, True, *args)
    else:
        spec = N.DropSpec(N.SAIT_DROP_THRESHOLD_CAP, args[0], args[1], 0, 0, args[2])
        expect = port.sait_thr_cap(T, True, *args)
    dT = S.DeviceCsr.upload(Tp)
    b = row_bounds(T.nrows, world)
    sess = []
    for q in range(world):
        h = C.c_void_p()
        N.check(N.lib.sait_build_session_create(dT.handle, 1, C.byref(spec), b[q], b[q + 1], None, C.byref(h)))
        sess.append(h)
    while N.lib.sait_build_session_remaining(sess[0]) > 0:
        flags = []
        for h in sess:
            ch = C.c_int(1)
            N.check(N.lib.sait_build_session_step(h, C.byref(ch)))
            flags.append(ch.value)
        if max(flags) == 0:
            for h in sess:
                N.check(N.lib.sait_build_session_stop(h))
    blocks = []
    for h in sess:
        out = C.c_void_p()
        N.check(N.lib.sait_build_session_finish(h, 1, C.byref(out), None))
        N.lib.sait_build_session_destroy(h)
        blocks.append(S.DeviceCsr(out.value).to_host())
    m = _assemble_mt_blocks(blocks, T.nrows)
    assert np.array_equal(m.indptr, expect.row_ptr) and np.array_equal(m.indices, expect.col_idx)
    assert bitwise_equal(m.data, expect.values)


def test_sharded_pair_world1_and_build_sharded_world1(S, golden):
    import torch

    from paper_2106_12836_b200 import _native as N
    from paper_2106_12836_b200.dist import ShardedPair, build_sharded

    ML, MU = to_product(golden_csr(golden, "c1/ML")), to_product(golden_csr(golden, "c1/MU"))
    sp = ShardedPair(ML, MU, 0, 1)
    r = torch.from_numpy(golden["c1/r"]).cuda()
    z = torch.empty_like(r)
    sp.apply(r, z)
    torch.cuda.synchronize()
    assert bitwise_equal(z.cpu().numpy(), golden["c1/z"])
    L = S.DeviceCsr.upload(to_product(golden_csr(golden, "c1/L")))
    spec = N.DropSpec(N.SAIT_DROP_THRESHOLD, 1e-2, 4, 0, 0, 0.0)
    blk, st, (c0, c1) = build_sharded(L, True, spec, 0, 1, transposed=False)
    assert (c0, c1) == (0, 4096) and st.steps_run == 4
    assert bitwise_equal_csr(blk.to_host(), golden_csr(golden, "c1/ML"))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _build_worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2106_12836_b200 as S
        from paper_2106_12836_b200 import _native as N
        from paper_2106_12836_b200.dist import build_sharded
        from oracle import oracle as O

        T = O.synthetic_lower(4000, 10, 0.005, seed=21)
        dT = S.DeviceCsr.upload(S.CsrMatrix(T.nrows, T.ncols, T.row_ptr, T.col_idx, T.values))
        spec = N.DropSpec(N.SAIT_DROP_THRESHOLD, 2e-2, 5, 0, 0, 0.0)
        blk, st, _ = build_sharded(dT, True, spec, rank, world)
        h = blk.to_host()
        np.savez(os.path.join(out_dir, f"blk{rank}.npz"), rp=h.row_ptr, ci=h.col_idx, v=h.values, n=h.ncols,
                 steps=st.steps_run)
    finally:
        dist.destroy_process_group()


def test_build_sharded_two_processes(tmp_path, S, port):
    import torch.multiprocessing as mp

    from oracle import oracle as O

    mp.start_processes(_build_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    blocks, steps = [], []
    for q in range(2):
        d = np.load(tmp_path / f"blk{q}.npz")
        blocks.append(S.CsrMatrix(len(d["rp"]) - 1, int(d["n"]), d["rp"], d["ci"], d["v"]))
        steps.append(int(d["steps"]))
    T = O.synthetic_lower(4000, 10, 0.005, seed=21)
    expect, nsteps = port.sait_thr_steps(T, True, 2e-2, 5)
    m = _assemble_mt_blocks(blocks, 4000)
    assert steps == [nsteps, nsteps]
    assert np.array_equal(m.indptr, expect.row_ptr) and np.array_equal(m.indices, expect.col_idx)
    assert bitwise_equal(m.data, expect.values)


@pytest.mark.parametrize("world,grid", [(2, 24), (3, 20), (4, 16)])
def test_peer_sharded_pair_virtual_ranks(S, port, world, grid):
    """PeerShardedPair's data path on one GPU: `world` ranks in one process,
    each reading its halo from the other ranks' buffers inside the SpMV.  The
    stages run rank by rank on one stream, so every flag a kernel waits on is
    already published (no cross-rank waiting on one GPU).  Three epochs
    exercise both parity copies; each rank's z rows equal the oracle's."""
    import torch

    from helpers import to_oracle
    from paper_2106_12836_b200.dist import PeerShardedPair

    A = S.laplacian_3d(grid)
    f = S.ilu_k(A, 0)
    ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
    ranks = {}
    resolve = lambda q, fac: ranks[q].bufs[fac].ptr  # noqa: E731
    for q in range(world):
        ranks[q] = PeerShardedPair(ML, MU, q, world, resolve=resolve)
    s = torch.cuda.current_stream().cuda_stream
    for epoch in (1, 2, 3):
        r = S.uniform_pm1(100 + epoch, A.nrows)
        want = port.pair_apply(to_oracle(ML), to_oracle(MU), r)
        rd = torch.from_numpy(r).cuda()
        zs = {}
        for q in range(world):
            a, b = ranks[q].own
            ranks[q].stage_input(rd[a:b], epoch, s)
        for q in range(world):
            ranks[q].stage_lower(epoch, s)
        for q in range(world):
            a, b = ranks[q].own
            zs[q] = torch.empty(b - a, dtype=torch.float64, device="cuda")
            ranks[q].stage_upper(zs[q], epoch, s)
        torch.cuda.synchronize()
        z = torch.cat([zs[q] for q in range(world)]).cpu().numpy()
        assert bitwise_equal(z, want), epoch
    assert all(ranks[q].halo_bytes > 0 for q in range(world))
    for q in range(world):
        ranks[q].close()


def test_peer_sharded_pair_world1(S, golden):
    """One rank: no halo, apply() equals the pair."""
    import torch

    from paper_2106_12836_b200.dist import PeerShardedPair

    ML, MU = to_product(golden_csr(golden, "c1/ML")), to_product(golden_csr(golden, "c1/MU"))
    P = PeerShardedPair(ML, MU, 0, 1, resolve=lambda q, f: None)
    r = torch.from_numpy(golden["c1/r"]).cuda()
    z = torch.empty_like(r)
    for _ in range(2):
        P.apply(r, z)
    torch.cuda.synchronize()
    assert bitwise_equal(z.cpu().numpy(), golden["c1/z"])
    P.close()


def _ipc_worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_12836_b200.dist import _DevBuf, _open_ipc
        from paper_2106_12836_b200 import _native as N

        n = 1 << 16
        buf = _DevBuf(8 * n + 256)
        buf.tensor(0, n).copy_(torch.arange(n, dtype=torch.float64, device="cuda") * (rank + 1))
        torch.cuda.synchronize()
        handles = [None] * world
        dist.all_gather_object(handles, buf.handle())
        peer = (rank + 1) % world
        ptr = _open_ipc(handles[peer])
        view = _DevBuf(8 * n, ptr=ptr, owned=False).tensor(0, n)
        got = view.cpu().numpy()
        dist.barrier()
        N.check(N.lib.sait_ipc_close(C.c_void_p(ptr)))
        np.save(os.path.join(out_dir, f"ipc{rank}.npy"), got)
        dist.barrier()
        buf.free()
    finally:
        dist.destroy_process_group()


def test_ipc_handles_two_processes(tmp_path):
    """The IPC plumbing of PeerShardedPair.distributed: each process exports a
    sait_device_alloc buffer, opens its peer's and reads the peer's values
    (two processes on one GPU; nothing waits on the other process's kernels)."""
    import torch.multiprocessing as mp

    mp.start_processes(_ipc_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    n = 1 << 16
    for q in range(2):
        got = np.load(tmp_path / f"ipc{q}.npy")
        assert np.array_equal(got, np.arange(n, dtype=np.float64) * (((q + 1) % 2) + 1))


def _virtual_sharded_build(S, T_dev, lower, spec, world, bounds):
    """Column-sharded build of `world` virtual ranks on one GPU with the global
    early stop reduced in-process; returns each rank's M[:, C_r:C_r+1]."""
    from paper_2106_12836_b200 import _native as N

    sess = []
    for q in range(world):
        h = C.c_void_p()
        N.check(N.lib.sait_build_session_create(T_dev.handle, int(lower), C.byref(spec), bounds[q], bounds[q + 1],
                                                None, C.byref(h)))
        sess.append(h)
    while N.lib.sait_build_session_remaining(sess[0]) > 0:
        flags = []
        for h in sess:
            ch = C.c_int(1)
            N.check(N.lib.sait_build_session_step(h, C.byref(ch)))
            flags.append(ch.value)
        if max(flags) == 0:
            for h in sess:
                N.check(N.lib.sait_build_session_stop(h))
    blocks = []
    for h in sess:
        out = C.c_void_p()
        N.check(N.lib.sait_build_session_finish(h, 0, C.byref(out), None))
        N.lib.sait_build_session_destroy(h)
        blocks.append(S.DeviceCsr(out.value))
    return blocks


@pytest.mark.parametrize("world,grid", [(2, 24), (3, 20), (4, 16)])
def test_sharded_build_redistribute_peer_apply_virtual_ranks(S, port, world, grid):
    """The device pipeline bench.py --gpus N runs, on one GPU with virtual
    ranks: column-sharded SAIT builds of both ILU factors with work-balanced
    column blocks (sait_column_work) -> column blocks redistributed to the
    apply's row blocks on the device (row_pieces + sait_csr_assemble_rows) ->
    PeerShardedPair.from_row_blocks.  Every row block equals the global
    factor's rows bitwise, and the peer-halo apply equals the oracle's pair
    apply over three epochs."""
    import torch

    from helpers import to_oracle
    from paper_2106_12836_b200 import _native as N
    from paper_2106_12836_b200.dist import (PeerShardedPair, column_bounds_by_work, redistribute_local,
                                            row_block_span, row_bounds)

    A = S.laplacian_3d(grid)
    f = S.ilu_k(A, 0)
    ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
    spec = N.DropSpec(N.SAIT_DROP_THRESHOLD, 5e-2, 3, 0, 0, 0.0)
    n = A.nrows
    rb = row_bounds(n, world)
    rows = []
    for lower, T, M in ((True, f.lower, ML), (False, f.upper, MU)):
        dT = S.DeviceCsr.upload(T)
        cb = column_bounds_by_work(dT, world)
        assert cb[0] == 0 and cb[-1] == n
        blocks = _virtual_sharded_build(S, dT, lower, spec, world, cb)
        rblocks = redistribute_local(blocks, cb, rb)
        for q in range(world):
            h = rblocks[q].to_host()
            a, b = M.row_ptr[rb[q]], M.row_ptr[rb[q + 1]]
            assert np.array_equal(h.row_ptr, M.row_ptr[rb[q]:rb[q + 1] + 1] - a)
            assert np.array_equal(h.col_idx, M.col_idx[a:b])
            assert bitwise_equal(h.values, M.values[a:b])
        rows.append(rblocks)
    spans = [[row_block_span(rows[f_][q], rb[q], rb[q + 1]) for q in range(world)] for f_ in range(2)]
    ranks = {}
    resolve = lambda q, fac: ranks[q].bufs[fac].ptr  # noqa: E731
    for q in range(world):
        ranks[q] = PeerShardedPair.from_row_blocks(rows[0][q], rows[1][q], spans[0], spans[1], rb, q, world,
                                                   resolve=resolve)
    s = torch.cuda.current_stream().cuda_stream
    for epoch in (1, 2, 3):
        r = S.uniform_pm1(300 + epoch, n)
        want = port.pair_apply(to_oracle(ML), to_oracle(MU), r)
        rd = torch.from_numpy(r).cuda()
        zs = {}
        for q in range(world):
            a, b = ranks[q].own
            ranks[q].stage_input(rd[a:b], epoch, s)
        for q in range(world):
            ranks[q].stage_lower(epoch, s)
        for q in range(world):
            a, b = ranks[q].own
            zs[q] = torch.empty(b - a, dtype=torch.float64, device="cuda")
            ranks[q].stage_upper(zs[q], epoch, s)
        torch.cuda.synchronize()
        z = torch.cat([zs[q] for q in range(world)]).cpu().numpy()
        assert bitwise_equal(z, want), epoch
    for q in range(world):
        ranks[q].close()


def test_column_work_matches_host(S):
    """sait_column_work: column j's predicted products (sum over the entries
    (k, j), k != j, of nnz(column k without its diagonal) + 1), against numpy."""
    import torch

    from oracle import oracle as O
    from paper_2106_12836_b200 import _native as N

    T = O.synthetic_lower(5000, 8, 0.01, seed=5)
    dT = S.DeviceCsr.upload(to_product(T))
    work = torch.empty(T.nrows, dtype=torch.int64, device="cuda")
    N.check(N.lib.sait_column_work(dT.handle, work.data_ptr(), None))
    rows = np.repeat(np.arange(T.nrows), np.diff(T.row_ptr))
    off = rows != T.col_idx
    cnt = np.bincount(T.col_idx[off], minlength=T.nrows)
    want = np.bincount(T.col_idx[off], weights=(cnt[rows[off]] + 1), minlength=T.nrows).astype(np.int64)
    assert np.array_equal(work.cpu().numpy(), want)


_NATIVE_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import torch
import paper_2106_12836_b200 as S
from paper_2106_12836_b200.dist import PeerShardedPair
from helpers import to_oracle
from oracle import oracle as O
P = O.get("port")
world = {world}
A = S.laplacian_3d(16)
f = S.ilu_k(A, 0)
ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
ranks = {{}}
resolve = lambda q, fac: ranks[q].bufs[fac].ptr
for q in range(world):
    ranks[q] = PeerShardedPair(ML, MU, q, world, resolve=resolve, align=256)
for q in range(world):
    ranks[q]._native_pair()  # created up front: creation synchronises the device (no waiting kernels queued yet)
streams = [torch.cuda.Stream() for _ in range(world)]
zs = {{q: torch.empty(ranks[q].own[1] - ranks[q].own[0], dtype=torch.float64, device="cuda") for q in range(world)}}
torch.cuda.synchronize()
ok = []
for epoch in (1, 2, 3, 4):
    r = S.uniform_pm1(500 + epoch, A.nrows)
    want = P.pair_apply(to_oracle(ML), to_oracle(MU), r)
    rd = torch.from_numpy(r).cuda()
    torch.cuda.synchronize()
    # nothing but the applies between here and the synchronize below: an
    # allocation or any call that synchronises the device would wait for
    # rank 0's kernels, which wait for rank 1's, which are not queued yet
    for q in range(world):
        a, b = ranks[q].own
        with torch.cuda.stream(streams[q]):
            ranks[q].apply(rd[a:b], zs[q])
    torch.cuda.synchronize()
    z = torch.cat([zs[q] for q in range(world)]).cpu().numpy()
    ok.append(int(np.array_equal(z.view(np.uint64), want.view(np.uint64))))
print(*ok)
for q in range(world):
    ranks[q].close()
"""


@pytest.mark.parametrize("world", [2, 3])
def test_native_peer_pair_concurrent_virtual_ranks(world):
    """The native peer-halo pair (sait_peer_pair_apply: boundary-slice copy +
    publish kernel, M_L reading its own x from r and publishing flag_U from
    its last CTA, M_U as a programmatic dependent) with `world` virtual ranks
    on one GPU, each on its own stream, so ranks really wait on each other's
    flags.  A 16^3 problem keeps every grid small enough (tens of CTAs) that
    all ranks' kernels are resident together; the child process is bounded
    by a timeout.  Four epochs (both parities twice) equal the oracle."""
    import subprocess
    import sys

    code = _NATIVE_CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"), world=world)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert out.stdout.split() == ["1", "1", "1", "1"]
