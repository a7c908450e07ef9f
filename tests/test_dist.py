"""Multi-process (gloo, CPU) tests of the multi-GPU host logic: halo plans and
the row-sharded pair apply.  Each rank computes its local SpMVs with the
oracle's CPU spmv (bitwise the reference's), exchanges halos over gloo, and
the gathered result must equal the un-sharded pair apply bit for bit."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, golden_csr


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class CpuOperator:
    def __init__(self, block):
        from oracle import oracle as O

        self.port = O.get("port")
        self.m = O.Csr(block.nrows, block.ncols, block.row_ptr, block.col_idx, block.values)

    def apply(self, x, y):
        import torch

        y.copy_(torch.from_numpy(self.port.spmv(self.m, x.numpy())))


def _worker(rank, world, port, case, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_12836_b200.csr import CsrMatrix
        from paper_2106_12836_b200.dist import ShardedPair

        data = np.load(case)
        ML = CsrMatrix(int(data["n"]), int(data["n"]), data["lrp"], data["lci"], data["lv"])
        MU = CsrMatrix(int(data["n"]), int(data["n"]), data["urp"], data["uci"], data["uv"])
        sp = ShardedPair(ML, MU, rank, world, make_operator=CpuOperator, device="cpu")
        r0, r1 = sp.own
        r = torch.from_numpy(data["r"][r0:r1].copy())
        z = torch.zeros(r1 - r0, dtype=torch.float64)
        for _ in range(2):  # buffers are reused across applies
            sp.apply(r, z)
        np.save(os.path.join(out_dir, f"z{rank}.npy"), z.numpy())
        np.save(os.path.join(out_dir, f"own{rank}.npy"), np.array(sp.own))
    finally:
        dist.destroy_process_group()


def _run(tmp_path, ML, MU, r, world):
    import torch.multiprocessing as mp

    case = str(tmp_path / "case.npz")
    np.savez(case, n=ML.nrows, lrp=ML.row_ptr, lci=ML.col_idx, lv=ML.values, urp=MU.row_ptr, uci=MU.col_idx,
             uv=MU.values, r=r)
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    z = np.zeros(ML.nrows)
    for q in range(world):
        a, b = np.load(tmp_path / f"own{q}.npy")
        z[a:b] = np.load(tmp_path / f"z{q}.npy")
    return z


def test_plans_cover_halos():
    from paper_2106_12836_b200.dist import make_plans, row_bounds

    b = row_bounds(5000, 4)
    assert b[0] == 0 and b[-1] == 5000 and all(x % 256 == 0 for x in b[:-1])
    spans = [(0, 1280), (100, 2560), (1000, 3840), (3800, 5000)]
    plans = make_plans(spans, b)
    for p in plans:
        covered = set(range(p.own[0], p.own[1]))
        for _, g0, g1 in p.recv:
            covered |= set(range(g0, g1))
        assert covered == set(range(p.lo, p.hi))
    sends = sorted((p.rank, q, g0, g1) for p in plans for (q, g0, g1) in p.send)
    recvs = sorted((q, p.rank, g0, g1) for p in plans for (q, g0, g1) in p.recv)
    assert sends == recvs
    assert plans[2].recv == [(0, 1000, 1280), (1, 1280, 2560)]  # halo spanning two ranks


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_apply_config1_bitwise(tmp_path, golden, port, world):
    from helpers import bitwise_equal

    ML, MU = golden_csr(golden, "c1/ML"), golden_csr(golden, "c1/MU")
    z = _run(tmp_path, ML, MU, golden["c1/r"], world)
    assert bitwise_equal(z, golden["c1/z"])


def test_sharded_apply_long_range_halo(tmp_path, port):
    """Config 4-like geometric offsets: the lower factor reaches across several
    ranks, so halos come from more than one peer."""
    from helpers import bitwise_equal
    from oracle import oracle as O

    T = O.synthetic_lower(2000, 6, 0.002, seed=9)
    ML = port.sait_thr(T, True, 5e-2, 3)
    MU = port.transpose(port.sait_thr(T, True, 1e-1, 2))
    r = O.uniform_pm1(3, 2000)
    z = _run(tmp_path, ML, MU, r, 4)
    assert bitwise_equal(z, port.pair_apply(ML, MU, r))


def _gather_worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_12836_b200.dist_solvers import TorchComm

        nb = 3 + 2 * rank  # ragged: the last rank of a sharded vector has fewer blocks
        mine = torch.arange(2 * nb, dtype=torch.float64).reshape(2, nb) + 100 * rank
        got = TorchComm(world).gather([mine])
        np.save(os.path.join(out_dir, f"g{rank}.npy"), torch.cat(got, dim=1).numpy())
    finally:
        dist.destroy_process_group()


def test_torchcomm_gathers_ragged_partials_in_rank_order(tmp_path):
    """dist_solvers.TorchComm: every rank receives all ranks' dot partials in
    rank order with their own lengths (the fold then matches one device)."""
    import torch.multiprocessing as mp

    mp.start_processes(_gather_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True,
                       start_method="spawn")
    want = np.concatenate([np.arange(2 * (3 + 2 * q), dtype=np.float64).reshape(2, -1) + 100 * q for q in range(3)],
                          axis=1)
    for q in range(3):
        assert np.array_equal(np.load(tmp_path / f"g{q}.npy"), want)


def _agree_worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_12836_b200.dist import _agree

        class Closable:
            closed = False

            def close(self):
                self.closed = True

        _agree(None, "ok", cleanup=None)  # nobody failed: returns on every rank
        obj = Closable()
        try:
            _agree(ValueError("no peer access") if rank == 1 else None, "PeerShardedPair", cleanup=obj)
            msg = "returned"
        except RuntimeError as exc:
            msg = str(exc)
        with open(os.path.join(out_dir, f"a{rank}.txt"), "w") as fh:
            fh.write(f"{msg}|{obj.closed}")
    finally:
        dist.destroy_process_group()


def test_multiprocess_construction_fails_together(tmp_path):
    """dist._agree: when one rank's peer-memory setup fails, EVERY rank raises
    (naming the failing rank) and releases what it built, so callers such as
    bench.py fall back to NCCL together instead of hanging in a collective."""
    import torch.multiprocessing as mp

    mp.start_processes(_agree_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    for q in range(2):
        msg, closed = (tmp_path / f"a{q}.txt").read_text().split("|")
        assert "construction failed on rank 1" in msg and "no peer access" in msg
        assert closed == "True"


def _host_pieces(block_rp, block_ci, block_v, row_bounds):
    """CPU stand-in of dist.row_pieces for a host block (test only)."""
    import torch

    out = []
    for q in range(len(row_bounds) - 1):
        r0, r1 = row_bounds[q], row_bounds[q + 1]
        a, b = int(block_rp[r0]), int(block_rp[r1])
        out.append({"nnz": b - a, "nrows": r1 - r0, "rp": torch.from_numpy(block_rp[r0:r1 + 1].astype(np.int32)),
                    "ci": torch.from_numpy(block_ci[a:b].astype(np.int32)), "v": torch.from_numpy(block_v[a:b].copy())})
    return out


def _host_assemble(pieces, col_bounds, nloc):
    """numpy restatement of sait_csr_assemble_rows (test only)."""
    rows_c, rows_v = [[] for _ in range(nloc)], [[] for _ in range(nloc)]
    for r in sorted(pieces):
        p = pieces[r]
        rp = p["rp"].numpy().astype(np.int64)
        rp = rp - rp[0]
        ci, v = p["ci"].numpy(), p["v"].numpy()
        for i in range(nloc):
            rows_c[i].extend((ci[rp[i]:rp[i + 1]] + col_bounds[r]).tolist())
            rows_v[i].extend(v[rp[i]:rp[i + 1]].tolist())
    rp = np.zeros(nloc + 1, dtype=np.int64)
    rp[1:] = np.cumsum([len(c) for c in rows_c])
    return rp, np.array(sum(rows_c, []), dtype=np.int64), np.array(sum(rows_v, []), dtype=np.float64)


def _redist_worker(rank, world, port, case, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2106_12836_b200.dist import exchange_row_pieces

        d = np.load(case)
        cb, rb = [int(x) for x in d["cb"]], [int(x) for x in d["rb"]]
        # this rank's column block M[:, C_r:C_r+1] (all n rows, local columns)
        mine = _host_pieces(d[f"rp{rank}"], d[f"ci{rank}"], d[f"v{rank}"], rb)
        nloc = rb[rank + 1] - rb[rank]
        got = exchange_row_pieces(mine, nloc, rank, world, device="cpu")
        rp, ci, v = _host_assemble(got, cb, nloc)
        np.savez(os.path.join(out_dir, f"rows{rank}.npz"), rp=rp, ci=ci, v=v)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_column_blocks_to_row_blocks(tmp_path, port, world):
    """dist.exchange_row_pieces (the K4 redistribution's transport, SURVEY.md
    §8e): every rank holds a column block M[:, C_r:C_{r+1}] of a SAIT factor
    (column bounds from the work balancer, row bounds of the apply); after the
    point-to-point exchange and the assembly rule of sait_csr_assemble_rows,
    each rank's rows equal the global factor's rows bitwise."""
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from paper_2106_12836_b200.dist import _bounds_from_work, row_bounds

    T = O.synthetic_lower(3000, 6, 0.01, seed=11)
    M = port.sait_thr(T, True, 1e-2, 3)
    n = M.nrows
    Mt = port.transpose(M)  # rows of M^T = columns of M
    work = np.diff(Mt.row_ptr) ** 2 + 1  # any positive weights
    cb = _bounds_from_work(work, world)
    assert cb[0] == 0 and cb[-1] == n and all(a <= b for a, b in zip(cb, cb[1:]))
    rb = row_bounds(n, world)
    arrays = {"cb": np.array(cb), "rb": np.array(rb)}
    for r in range(world):
        # M[:, c0:c1] as an n-row CSR with local columns (what build_sharded returns)
        a, b = cb[r], cb[r + 1]
        rows = [[(c - a, v) for c, v in zip(M.col_idx[M.row_ptr[i]:M.row_ptr[i + 1]],
                                           M.values[M.row_ptr[i]:M.row_ptr[i + 1]]) if a <= c < b] for i in range(n)]
        rp = np.zeros(n + 1, dtype=np.int64)
        rp[1:] = np.cumsum([len(x) for x in rows])
        arrays[f"rp{r}"] = rp
        arrays[f"ci{r}"] = np.array([c for x in rows for c, _ in x], dtype=np.int64)
        arrays[f"v{r}"] = np.array([v for x in rows for _, v in x], dtype=np.float64)
    case = str(tmp_path / "case.npz")
    np.savez(case, **arrays)
    mp.start_processes(_redist_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    for q in range(world):
        got = np.load(tmp_path / f"rows{q}.npz")
        r0, r1 = rb[q], rb[q + 1]
        a, b = M.row_ptr[r0], M.row_ptr[r1]
        assert np.array_equal(got["rp"], M.row_ptr[r0:r1 + 1] - a)
        assert np.array_equal(got["ci"], M.col_idx[a:b])
        assert np.array_equal(got["v"].view(np.uint64), M.values[a:b].view(np.uint64))


def test_work_balanced_bounds():
    """Column blocks cut on the prefix sums of the predicted work: every block
    carries at most its share plus one column's work."""
    from paper_2106_12836_b200.dist import _bounds_from_work

    rng = np.random.default_rng(3)
    w = rng.integers(1, 50, 10000)
    w[:20] = 5000  # heavy first columns (C4's capped offsets pile onto them)
    for world in (1, 2, 4, 8):
        b = _bounds_from_work(w, world)
        assert len(b) == world + 1 and b[0] == 0 and b[-1] == len(w)
        share = w.sum() / world
        for r in range(world):
            assert w[b[r]:b[r + 1]].sum() <= share + w.max()
