"""Multi-GPU plumbing: row-sharded SAIT apply with halo
exchange, column-sharded SAIT build with a global early-stop reduction.

One process per GPU; ``torch.distributed`` carries the data (NCCL over
NVLink on B200, gloo in the CPU tests).  The kernels are the single-GPU ones
(``sait_operator_*`` / ``sait_build_session_*`` in the C ABI).

Apply.  Rank r owns rows [R_r, R_{r+1}) of both factors and of r, y, z.
The columns its rows of a factor touch form one contiguous range; its local
factor block is re-indexed into an extended vector ``[halo below | own |
halo above]``.  Before M_L the missing r entries are received from the ranks
that own them, before M_U the missing y entries — the only data-path
communication.  For the banded SAIT factors the halo is one bandwidth
(n^2 + n rows for an n^3 stencil) from the neighbouring rank(s).

Build.  A column of M evolves independently, so rank r
runs the recursion on the rows [C_r, C_{r+1}) of M^T; after each step the
ranks all-reduce (MAX) their "changed" flag, keeping the reference's global
early stop (sait.cpp:84-85) and therefore its step count and bits.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

GROUP_ROWS = 256


def row_bounds(n: int, world: int, align: int = GROUP_ROWS) -> list[int]:
    """world + 1 boundaries splitting [0, n) into near-equal, aligned blocks."""
    per = -(-n // world)
    per = -(-per // align) * align
    return [min(n, r * per) for r in range(world)] + [n]


def column_span(row_ptr: np.ndarray, col_idx: np.ndarray, r0: int, r1: int) -> tuple[int, int]:
    """[lo, hi) of the columns the rows [r0, r1) touch ((r0, r0) if none)."""
    b, e = int(row_ptr[r0]), int(row_ptr[r1])
    if e <= b:
        return r0, r0
    seg = col_idx[b:e]
    return int(seg.min()), int(seg.max()) + 1


@dataclass
class HaloPlan:
    rank: int
    own: tuple[int, int]                 # rows owned (global)
    lo: int                              # extended vector covers [lo, hi)
    hi: int
    recv: list[tuple[int, int, int]] = field(default_factory=list)  # (peer, g0, g1) into ext
    send: list[tuple[int, int, int]] = field(default_factory=list)  # (peer, g0, g1) from own

    @property
    def ext_len(self) -> int:
        return self.hi - self.lo

    @property
    def own_offset(self) -> int:
        return self.own[0] - self.lo


def make_plans(spans: list[tuple[int, int]], bounds: list[int]) -> list[HaloPlan]:
    """Plans for every rank from every rank's column span (deterministic, so
    each rank can compute all of them without communication)."""
    world = len(bounds) - 1
    plans = []
    for r in range(world):
        r0, r1 = bounds[r], bounds[r + 1]
        lo, hi = spans[r]
        lo, hi = min(lo, r0), max(hi, r1)
        plans.append(HaloPlan(r, (r0, r1), lo, hi))
    for r, p in enumerate(plans):
        for q in range(world):
            if q == r:
                continue
            g0, g1 = max(p.lo, bounds[q]), min(p.hi, bounds[q + 1])
            if g1 > g0:
                p.recv.append((q, g0, g1))
                plans[q].send.append((r, g0, g1))
    for p in plans:  # deterministic order: by peer
        p.recv.sort()
        p.send.sort()
    return plans


def local_block(row_ptr, col_idx, values, r0: int, r1: int, lo: int, ext_len: int):
    """Rows [r0, r1) of a global CSR with columns shifted by -lo: a
    (r1 - r0) x ext_len host CSR (reference layout)."""
    from .csr import CsrMatrix

    b, e = int(row_ptr[r0]), int(row_ptr[r1])
    rp = np.asarray(row_ptr[r0 : r1 + 1], dtype=np.int64) - b
    ci = np.asarray(col_idx[b:e], dtype=np.int64) - lo
    return CsrMatrix(r1 - r0, ext_len, rp, ci, np.asarray(values[b:e], dtype=np.float64))


def exchange(ext, own, plan: HaloPlan, group=None) -> None:
    """Fill ext's halo slices from their owners; send our own slices.
    ``ext`` / ``own`` are 1-D torch tensors (CUDA with NCCL, CPU with gloo)."""
    import torch.distributed as dist

    reqs = []
    for peer, g0, g1 in plan.recv:
        reqs.append(dist.irecv(ext[g0 - plan.lo : g1 - plan.lo], src=peer, group=group))
    for peer, g0, g1 in plan.send:
        s0 = g0 - plan.own[0]
        reqs.append(dist.isend(own[s0 : s0 + (g1 - g0)].contiguous(), dst=peer, group=group))
    for q in reqs:
        q.wait()


class DeviceOperator:
    """y = A x for a local block on the current GPU (sait_operator_*)."""

    def __init__(self, block):
        from . import _native as N
        from .csr import DeviceCsr

        d = DeviceCsr.upload(block)
        h = C.c_void_p()
        N.check(N.lib.sait_operator_create(d.handle, 1, C.byref(h)))
        d.release()
        self._h = h
        self.nrows, self.ncols = block.nrows, block.ncols

    @classmethod
    def from_device(cls, d):
        """From a device CSR (ownership moves into the operator)."""
        from . import _native as N

        obj = cls.__new__(cls)
        h = C.c_void_p()
        N.check(N.lib.sait_operator_create(d.handle, 1, C.byref(h)))
        d.release()
        obj._h = h
        obj.nrows, obj.ncols = d.nrows, d.ncols
        return obj

    def apply(self, x, y, stream=None):
        import torch

        from . import _native as N

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        N.check(N.lib.sait_operator_apply(self._h, x.data_ptr(), x.numel(), y.data_ptr(), y.numel(), s))

    def __del__(self):
        try:
            from . import _native as N

            N.lib.sait_operator_destroy(self._h)
        except Exception:
            pass


class ShardedPair:
    """Row-sharded z = M_U (M_L r): each rank passes its own rows of r and
    receives its own rows of z.  ``make_operator(block) -> obj.apply(x, y)``
    selects the compute backend (DeviceOperator on GPUs)."""

    def __init__(self, ML, MU, rank: int, world: int, group=None, make_operator=DeviceOperator, device="cuda"):
        import torch

        n = ML.nrows
        if not (ML.ncols == n and MU.nrows == n and MU.ncols == n):
            raise ValueError("ShardedPair: square factors of equal order required")
        self.n, self.rank, self.world, self.group = n, rank, world, group
        self.bounds = row_bounds(n, world)
        spans_l = [column_span(ML.row_ptr, ML.col_idx, self.bounds[q], self.bounds[q + 1]) for q in range(world)]
        spans_u = [column_span(MU.row_ptr, MU.col_idx, self.bounds[q], self.bounds[q + 1]) for q in range(world)]
        self.plan_l = make_plans(spans_l, self.bounds)[rank]
        self.plan_u = make_plans(spans_u, self.bounds)[rank]
        r0, r1 = self.bounds[rank], self.bounds[rank + 1]
        self.own = (r0, r1)
        self.op_l = make_operator(local_block(ML.row_ptr, ML.col_idx, ML.values, r0, r1, self.plan_l.lo, self.plan_l.ext_len))
        self.op_u = make_operator(local_block(MU.row_ptr, MU.col_idx, MU.values, r0, r1, self.plan_u.lo, self.plan_u.ext_len))
        kw = dict(dtype=torch.float64, device=device)
        self.ext_l = torch.zeros(self.plan_l.ext_len, **kw)
        self.ext_u = torch.zeros(self.plan_u.ext_len, **kw)
        self.halo_bytes = 8 * sum(g1 - g0 for _, g0, g1 in self.plan_l.recv + self.plan_u.recv)

    def apply(self, r_local, z_local) -> None:
        pl, pu = self.plan_l, self.plan_u
        nloc = self.own[1] - self.own[0]
        own_l = self.ext_l[pl.own_offset : pl.own_offset + nloc]
        own_u = self.ext_u[pu.own_offset : pu.own_offset + nloc]
        own_l.copy_(r_local)
        exchange(self.ext_l, own_l, pl, self.group)
        self.op_l.apply(self.ext_l, own_u)        # y rows land in M_U's extended vector
        exchange(self.ext_u, own_u, pu, self.group)
        self.op_u.apply(self.ext_u, z_local)


def build_sharded(T_dev, lower: bool, spec, rank: int, world: int, group=None, stream=None, transposed: bool = True,
                  reduce_max=None, bounds: list[int] | None = None):
    """Column-sharded SAIT build: this rank's block of columns of M.

    Returns (DeviceCsr block, BuildStats, (c0, c1)).  ``transposed`` selects the
    rows of M^T (a (c1-c0) x n CSR) or M[:, c0:c1].  ``reduce_max(int) -> int``
    is the cross-rank reduction (all-reduce MAX over ``group`` by default)."""
    from . import _native as N
    from .csr import DeviceCsr, _stream_handle
    from .sait import BuildStats

    if reduce_max is None:
        reduce_max = _allreduce_max(group)
    n = T_dev.nrows
    if bounds is None:
        bounds = row_bounds(n, world)
    c0, c1 = bounds[rank], bounds[rank + 1]
    sh = _stream_handle(stream)
    sess = C.c_void_p()
    N.check(N.lib.sait_build_session_create(T_dev.handle, int(lower), C.byref(spec), c0, c1, sh, C.byref(sess)))
    try:
        while N.lib.sait_build_session_remaining(sess) > 0:
            ch = C.c_int(1)
            N.check(N.lib.sait_build_session_step(sess, C.byref(ch)))
            if reduce_max(int(ch.value)) == 0:  # no column block changed: global early stop
                N.check(N.lib.sait_build_session_stop(sess))
        out = C.c_void_p()
        st = N.BuildStats()
        N.check(N.lib.sait_build_session_finish(sess, int(transposed), C.byref(out), C.byref(st)))
    finally:
        N.lib.sait_build_session_destroy(sess)
    return DeviceCsr(out.value), BuildStats(st.steps_run, bool(st.stabilized), st.nnz_out, st.products, st.seconds), (c0, c1)


def column_bounds_by_work(T_dev, world: int, stream=None) -> list[int]:
    """world + 1 column boundaries for the column-sharded build, balanced on
    the predicted products per column (sait_column_work: column j's step-2
    work) rather than on the column count."""
    import torch

    from . import _native as N
    from .csr import _stream_handle

    n = T_dev.nrows
    work = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
    N.check(N.lib.sait_column_work(T_dev.handle, work.data_ptr(), s))
    return _bounds_from_work(work[:n].cpu().numpy(), world)


def _bounds_from_work(work: np.ndarray, world: int) -> list[int]:
    n = len(work)
    cum = np.cumsum(work, dtype=np.int64)
    total = int(cum[-1]) if n else 0
    b = [0]
    for r in range(1, world):
        j = int(np.searchsorted(cum, total * r / world, side="left")) + 1 if total else n * r // world
        b.append(min(n, max(b[-1], j)))
    b.append(n)
    return b


# ------------------------------------------ column blocks -> row blocks (K4)
# The column-sharded build leaves rank r with M[:, C_r:C_{r+1}] (all n rows,
# local columns); the row-sharded apply needs rows [R_q, R_{q+1}) of M on rank
# q.  Rank r cuts its block at the row bounds (one device read of n_ranks + 1
# row pointers), sends piece q to rank q (NCCL point-to-point: row pointers,
# columns, values), and rank q assembles its row block from the pieces in
# ascending r (sait_csr_assemble_rows: row i = the pieces' rows i
# concatenated, columns shifted by C_r -- sorted because the column blocks
# ascend).  The distributed form of transpose (csr.cpp:72-92); no host round
# trip of the matrix.

def _dev_view(ptr: int, count: int, dtype: str):
    import torch

    iface = {"shape": (count,), "typestr": dtype, "data": (ptr, False), "version": 3, "strides": None}
    holder = type("CudaArray", (), {"__cuda_array_interface__": iface})()
    return torch.as_tensor(holder, device="cuda")


def row_pieces(block, row_bounds: list[int], stream=None) -> list[dict]:
    """Rank-local cut of a device CSR block (n rows) at the row bounds: for
    every destination q its row pointers (rows R_q..R_{q+1}, not rebased),
    columns and values as device views, and its entry count."""
    import torch

    from . import _native as N
    from .csr import _stream_handle

    world = len(row_bounds) - 1
    s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
    rows = (C.c_int64 * (world + 1))(*row_bounds)
    offs = (C.c_int64 * (world + 1))()
    N.check(N.lib.sait_csr_row_ptr_at(block.handle, rows, world + 1, offs, s))
    rp, ci, v = block.device_arrays()
    out = []
    for q in range(world):
        r0, r1 = row_bounds[q], row_bounds[q + 1]
        nnz = int(offs[q + 1] - offs[q])
        out.append({"nnz": nnz, "nrows": r1 - r0,
                    "rp": _dev_view(rp + 4 * r0, r1 - r0 + 1, "<i4"),
                    "ci": _dev_view(ci + 4 * int(offs[q]), max(nnz, 1), "<i4")[:nnz],
                    "v": _dev_view(v + 8 * int(offs[q]), max(nnz, 1), "<f8")[:nnz]})
    return out


def exchange_row_pieces(mine: list[dict], nloc: int, rank: int, world: int, group=None, device="cuda") -> dict:
    """Send piece q of `mine` to rank q, receive every rank's piece of our rows
    (torch.distributed point-to-point, batched).  Returns {r: piece} for the
    ranks with entries for us (ours included, not copied)."""
    import torch
    import torch.distributed as dist

    counts = torch.tensor([p["nnz"] for p in mine], dtype=torch.int64, device=device)
    allc = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts, group=group)
    recv_cnt = [int(allc[r][rank]) for r in range(world)]
    ops, got = [], {}
    for q in range(world):
        p = mine[q]
        if q != rank and p["nnz"]:
            for t in (p["rp"], p["ci"], p["v"]):
                ops.append(dist.P2POp(dist.isend, t.contiguous(), q, group=group))
    for r in range(world):
        if r == rank or not recv_cnt[r]:
            continue
        b = {"nnz": recv_cnt[r], "nrows": nloc,
             "rp": torch.empty(nloc + 1, dtype=torch.int32, device=device),
             "ci": torch.empty(recv_cnt[r], dtype=torch.int32, device=device),
             "v": torch.empty(recv_cnt[r], dtype=torch.float64, device=device)}
        got[r] = b
        for t in (b["rp"], b["ci"], b["v"]):
            ops.append(dist.P2POp(dist.irecv, t, r, group=group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    if mine[rank]["nnz"]:
        got[rank] = mine[rank]
    return got


def assemble_row_block(pieces: dict, col_bounds: list[int], nloc: int, ncols: int, stream=None):
    """Device assembly (sait_csr_assemble_rows) of the pieces {r: piece} in
    ascending r, columns shifted by C_r."""
    import torch

    from . import _native as N
    from .csr import DeviceCsr, _stream_handle

    order = sorted(pieces)
    arr = (N.RowPiece * max(1, len(order)))()
    for k, r in enumerate(order):
        p = pieces[r]
        arr[k].row_ptr, arr[k].col_idx, arr[k].values = p["rp"].data_ptr(), p["ci"].data_ptr(), p["v"].data_ptr()
        arr[k].col_offset = int(col_bounds[r])
    s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
    h = C.c_void_p()
    N.check(N.lib.sait_csr_assemble_rows(len(order), arr, nloc, ncols, s, C.byref(h)))
    return DeviceCsr(h.value)


def redistribute_to_rows(block, col_bounds: list[int], row_bounds: list[int], rank: int, world: int, group=None,
                         stream=None):
    """This rank's rows [R_rank, R_rank+1) of M (global columns) from every
    rank's column block M[:, C_r:C_r+1] (see above)."""
    mine = row_pieces(block, row_bounds, stream)
    nloc = row_bounds[rank + 1] - row_bounds[rank]
    got = exchange_row_pieces(mine, nloc, rank, world, group)
    return assemble_row_block(got, col_bounds, nloc, block.nrows, stream)


def redistribute_local(blocks: list, col_bounds: list[int], row_bounds: list[int], stream=None) -> list:
    """The same for virtual ranks living in one process (one GPU): rank q's
    row block assembled straight from every block's piece q."""
    world = len(blocks)
    cuts = [row_pieces(b, row_bounds, stream) for b in blocks]
    out = []
    for q in range(world):
        pieces = {r: cuts[r][q] for r in range(world) if cuts[r][q]["nnz"]}
        out.append(assemble_row_block(pieces, col_bounds, row_bounds[q + 1] - row_bounds[q], blocks[0].nrows, stream))
    return out


def row_block_span(block, r0: int, r1: int, stream=None) -> tuple[int, int]:
    """Column span of a device row block (global columns), own rows included
    by make_plans."""
    import torch

    from . import _native as N
    from .csr import _stream_handle

    s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
    lo, hi = C.c_int64(), C.c_int64()
    N.check(N.lib.sait_csr_col_span(block.handle, C.byref(lo), C.byref(hi), s))
    if hi.value <= lo.value:
        return r0, r0
    return lo.value, hi.value


def _allreduce_max(group):
    def red(v: int) -> int:
        import torch
        import torch.distributed as dist

        if not dist.is_initialized():
            return v
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return int(t.item())

    return red


class _DevBuf:
    """A device buffer from sait_device_alloc (plain cudaMalloc, so CUDA IPC
    can export it), viewable as a torch tensor via __cuda_array_interface__."""

    def __init__(self, nbytes: int, ptr: int | None = None, owned: bool = True):
        from . import _native as N

        self.nbytes = nbytes
        self.owned = owned and ptr is None
        if ptr is None:
            p = C.c_void_p()
            N.check(N.lib.sait_device_alloc(nbytes, C.byref(p)))
            ptr = p.value
        self.ptr = ptr

    def tensor(self, offset_bytes: int, count: int, dtype: str = "<f8"):
        import torch

        itemsize = 8 if dtype == "<f8" else 4
        iface = {"shape": (count,), "typestr": dtype, "data": (self.ptr + offset_bytes, False), "version": 3,
                 "strides": None}
        holder = type("CudaArray", (), {"__cuda_array_interface__": iface})()
        del itemsize
        return torch.as_tensor(holder, device="cuda")

    def handle(self) -> bytes:
        from . import _native as N

        h = (C.c_char * 64)()
        N.check(N.lib.sait_ipc_handle(C.c_void_p(self.ptr), h))
        return bytes(h)

    def free(self):
        from . import _native as N

        if self.owned and self.ptr:
            N.lib.sait_device_free(C.c_void_p(self.ptr))
        self.ptr = 0


def _open_ipc(handle: bytes) -> int:
    from . import _native as N

    p = C.c_void_p()
    N.check(N.lib.sait_ipc_open(C.create_string_buffer(handle, 64), C.byref(p)))
    return p.value


class PeerShardedPair:
    """Row-sharded z = M_U (M_L r) with no collective on the data path: each
    rank's SpMV reads its halo straight from the neighbours' extended vectors
    (sait_operator_apply_halo over peer memory / NVLink), after the owner
    published the epoch (sait_publish_epoch).  Per factor every rank owns two
    parity copies of its extended vector [halo | own | halo] plus an epoch
    flag in one IPC-exportable allocation; an apply writes the own segment of
    copy (epoch & 1), so a neighbour still reading epoch e never sees e + 1's
    values (a rank cannot run two epochs ahead: each apply also needs its
    neighbours' values of the same epoch).

    ``resolve(rank, factor) -> device address`` gives another rank's buffer
    base: IPC-opened in a multi-process job (``distributed``), or the plain
    pointer when several ranks live in one process (the single-GPU test).
    Raises NotImplementedError when a halo spans more than one peer per side
    (use ShardedPair)."""

    def __init__(self, ML, MU, rank: int, world: int, resolve=None, align: int = GROUP_ROWS):
        n = ML.nrows
        if not (ML.ncols == n and MU.nrows == n and MU.ncols == n):
            raise ValueError("PeerShardedPair: square factors of equal order required")
        self.n, self.rank, self.world = n, rank, world
        self.bounds = row_bounds(n, world, align)
        self.plans = []
        for M in (ML, MU):
            spans = [column_span(M.row_ptr, M.col_idx, self.bounds[q], self.bounds[q + 1]) for q in range(world)]
            allp = make_plans(spans, self.bounds)
            for p in allp:
                below = [x for x in p.recv if x[2] <= p.own[0]]
                above = [x for x in p.recv if x[1] >= p.own[1]]
                if len(below) > 1 or len(above) > 1:
                    raise NotImplementedError("PeerShardedPair: a halo spans several ranks")
            self.plans.append(allp)
        r0, r1 = self.bounds[rank], self.bounds[rank + 1]
        ops = []
        for f, M in enumerate((ML, MU)):
            p = self.plans[f][rank]
            ops.append(DeviceOperator(local_block(M.row_ptr, M.col_idx, M.values, r0, r1, p.lo, p.ext_len)))
        self._setup(ops, resolve)

    def _setup(self, ops, resolve):
        rank = self.rank
        self.own = (self.bounds[rank], self.bounds[rank + 1])
        self.ops, self.bufs = ops, []
        for f in range(2):
            self.bufs.append(_DevBuf(self._buf_bytes(f, rank)))
            self.bufs[f].tensor(self._flag_off(f, rank), 1, "<i4").zero_()
        self.resolve = resolve
        self.epoch = 0
        self.halo_bytes = 8 * sum(g1 - g0 for f in range(2) for _, g0, g1 in self.plans[f][rank].recv)

    @classmethod
    def from_row_blocks(cls, bl, bu, spans_l, spans_u, bounds, rank: int, world: int, resolve=None):
        """From this rank's device row blocks of M_L and M_U (rows [R_rank,
        R_rank+1), global columns -- e.g. redistribute_to_rows of a
        column-sharded build) and every rank's column spans; the blocks are
        re-indexed in place into the extended vector and owned by the pair."""
        from . import _native as N

        obj = cls.__new__(cls)
        obj.n, obj.rank, obj.world = bounds[-1], rank, world
        obj.bounds = list(bounds)
        obj.plans = [make_plans(list(spans_l), obj.bounds), make_plans(list(spans_u), obj.bounds)]
        for allp in obj.plans:
            for p in allp:
                below = [x for x in p.recv if x[2] <= p.own[0]]
                above = [x for x in p.recv if x[1] >= p.own[1]]
                if len(below) > 1 or len(above) > 1:
                    raise NotImplementedError("PeerShardedPair: a halo spans several ranks")
        ops = []
        for f, blk in enumerate((bl, bu)):
            p = obj.plans[f][rank]
            N.check(N.lib.sait_csr_shift_cols(blk.handle, -p.lo, p.ext_len, None))
            blk.ncols = p.ext_len
            ops.append(DeviceOperator.from_device(blk))
        obj._setup(ops, resolve)
        return obj

    # layout of rank q's buffer for factor f: [ext parity 0 | ext parity 1 | flag]
    def _ext_len(self, f, q):
        return self.plans[f][q].ext_len

    def _buf_bytes(self, f, q):
        return 16 * self._ext_len(f, q) + 256

    def _flag_off(self, f, q):
        return 16 * self._ext_len(f, q) + 128

    def _halo(self, f, epoch):
        from . import _native as N

        p = self.plans[f][self.rank]
        par = epoch & 1
        h = N.Halo()
        h.own_lo, h.own_hi = p.own[0] - p.lo, p.own[1] - p.lo
        h.epoch = epoch
        for peer, g0, g1 in p.recv:
        # the peer's extended vector of the same parity; global g sits at g - lo_peer
            pq = self.plans[f][peer]
            base = self.resolve(peer, f) + 8 * par * pq.ext_len
            flag = self.resolve(peer, f) + self._flag_off(f, peer)
            if g1 <= p.own[0]:
                h.lo_src, h.lo_shift, h.lo_flag = base, p.lo - pq.lo, flag
            else:
                h.hi_src, h.hi_shift, h.hi_flag = base, p.lo - pq.lo, flag
        return h

    def _ext(self, f, par):
        return self.bufs[f].tensor(8 * par * self._ext_len(f, self.rank), self._ext_len(f, self.rank))

    def _own(self, f, par):
        p = self.plans[f][self.rank]
        return self._ext(f, par)[p.own_offset : p.own_offset + (self.own[1] - self.own[0])]

    def _publish(self, f, epoch, s):
        from . import _native as N

        flag = self.bufs[f].ptr + self._flag_off(f, self.rank)
        N.check(N.lib.sait_publish_epoch(C.c_void_p(flag), int(epoch), s))

    def _spmv(self, f, epoch, out, s):
        from . import _native as N

        x = self._ext(f, epoch & 1)
        h = self._halo(f, epoch)
        N.check(N.lib.sait_operator_apply_halo(self.ops[f]._h, x.data_ptr(), x.numel(), C.byref(h), out.data_ptr(),
                                               out.numel(), s))

    # the apply in three stages (a multi-rank single-process test interleaves them)
    def stage_input(self, r_local, epoch, s):
        self._own(0, epoch & 1).copy_(r_local)
        self._publish(0, epoch, s)

    def stage_lower(self, epoch, s):
        self._spmv(0, epoch, self._own(1, epoch & 1), s)  # y lands in M_U's extended vector
        self._publish(1, epoch, s)

    def stage_upper(self, z_local, epoch, s):
        self._spmv(1, epoch, z_local, s)

    def _native_pair(self):
        """The data path as one native object (sait_peer_pair_*).  Creating it
        synchronises the device, so it must exist before any apply that
        waits on a peer is queued (distributed() creates it eagerly; ranks
        living in one process create all of theirs first)."""
        from . import _native as N

        if getattr(self, "_pp", None) is None:
            desc = (N.PeerFactorDesc * 2)()
            for f in range(2):
                p = self.plans[f][self.rank]
                d = desc[f]
                d.ext[0] = self.bufs[f].ptr
                d.ext[1] = self.bufs[f].ptr + 8 * self._ext_len(f, self.rank)
                d.flag = self.bufs[f].ptr + self._flag_off(f, self.rank)
                d.ext_len, d.own_offset, d.own_len = p.ext_len, p.own_offset, self.own[1] - self.own[0]
                # own rows the neighbours read (at most one range per side)
                rng = sorted((g0 - self.own[0], g1 - g0) for _, g0, g1 in p.send)
                if len(rng) > 2:
                    raise NotImplementedError("PeerShardedPair: own rows read by more than two ranks")
                rng += [(0, 0)] * (2 - len(rng))
                (d.send_a0, d.send_n0), (d.send_a1, d.send_n1) = rng
                for par in range(2):
                    d.halo[par] = self._halo(f, par)
            h = C.c_void_p()
            N.check(N.lib.sait_peer_pair_create(self.ops[0]._h, self.ops[1]._h, desc, C.byref(h)))
            self._pp = h
        return self._pp

    def apply(self, r_local, z_local, stream=None) -> None:
        """z_local = (M_U M_L r)[own rows]; epochs advance inside the native
        object (do not mix with the stage_* calls)."""
        import torch

        from . import _native as N

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        N.check(N.lib.sait_peer_pair_apply(self._native_pair(), r_local.data_ptr(), z_local.data_ptr(), s))

    @classmethod
    def distributed(cls, ML, MU, rank: int, world: int, group=None, align: int = GROUP_ROWS):
        """Multi-process construction: the ranks swap IPC handles of their
        buffers (torch.distributed all_gather_object) and open their peers'."""
        return cls._connect(lambda: cls(ML, MU, rank, world, resolve=None, align=align), rank, world, group)

    @classmethod
    def distributed_from_row_blocks(cls, bl, bu, bounds, rank: int, world: int, group=None):
        """Multi-process construction from device row blocks (global columns):
        the column spans are all-gathered, then the IPC handles as above."""
        import torch.distributed as dist

        r0, r1 = bounds[rank], bounds[rank + 1]
        mine = (row_block_span(bl, r0, r1), row_block_span(bu, r0, r1))
        spans = [None] * world
        dist.all_gather_object(spans, mine, group=group)
        return cls._connect(lambda: cls.from_row_blocks(bl, bu, [x[0] for x in spans], [x[1] for x in spans], bounds,
                                                        rank, world), rank, world, group)

    @classmethod
    def _connect(cls, make, rank: int, world: int, group=None):
        import torch.distributed as dist

        obj, mine, err = None, None, None
        try:
            obj = make()
            mine = [obj.bufs[0].handle(), obj.bufs[1].handle()]
        except Exception as exc:  # noqa: BLE001  (agreed on below)
            err = exc
        _agree(err, "PeerShardedPair", group, cleanup=obj)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        opened = {}
        try:
            for f in range(2):
                for peer, _, _ in obj.plans[f][rank].recv:
                    opened[(peer, f)] = _open_ipc(allh[peer][f])
        except Exception as exc:  # noqa: BLE001
            err = exc
        obj._opened = opened
        _agree(err, "PeerShardedPair", group, cleanup=obj)
        obj.resolve = lambda q, f: obj.bufs[f].ptr if q == rank else opened[(q, f)]
        obj._native_pair()
        dist.barrier(group=group)
        return obj

    def close(self):
        from . import _native as N

        if getattr(self, "_pp", None) is not None:
            N.lib.sait_peer_pair_destroy(self._pp)
            self._pp = None
        for p in getattr(self, "_opened", {}).values():
            N.lib.sait_ipc_close(C.c_void_p(p))
        self._opened = {}
        for b in self.bufs:
            b.free()


def _agree(err, what, group=None, cleanup=None):
    """Collective error agreement for multi-process construction: every rank
    reaches this point, and if ANY rank failed, ALL of them raise (so callers
    fall back together instead of leaving peers blocked in a collective)."""
    import torch.distributed as dist

    mine = None if err is None else f"{type(err).__name__}: {err}"
    allerr = [None] * dist.get_world_size(group)
    dist.all_gather_object(allerr, mine, group=group)
    bad = [(q, e) for q, e in enumerate(allerr) if e is not None]
    if bad:
        if cleanup is not None:
            try:
                cleanup.close()
            except Exception:  # noqa: BLE001
                pass
        q, e = bad[0]
        raise RuntimeError(f"{what}: construction failed on rank {q}: {e}") from err


class PeerRowOperator:
    """Row block of one sharded matrix, y_local = (A x)_local, with the halo
    of x read from the neighbours' buffers inside the SpMV (the single-matrix
    form of PeerShardedPair: the system matrix of a sharded solver loop)."""

    def __init__(self, A, rank: int, world: int, resolve=None, align: int = GROUP_ROWS):
        n = A.nrows
        if A.ncols != n:
            raise ValueError("PeerRowOperator: square matrix required")
        self.n, self.rank, self.world = n, rank, world
        self.bounds = row_bounds(n, world, align)
        spans = [column_span(A.row_ptr, A.col_idx, self.bounds[q], self.bounds[q + 1]) for q in range(world)]
        self.plans = make_plans(spans, self.bounds)
        for p in self.plans:
            if len([x for x in p.recv if x[2] <= p.own[0]]) > 1 or len([x for x in p.recv if x[1] >= p.own[1]]) > 1:
                raise NotImplementedError("PeerRowOperator: a halo spans several ranks")
        r0, r1 = self.bounds[rank], self.bounds[rank + 1]
        if r1 <= r0:
            raise ValueError(f"PeerRowOperator: rank {rank} owns no rows (n={n}, world={world}, align={align})")
        self.own = (r0, r1)
        p = self.plans[rank]
        self.op = DeviceOperator(local_block(A.row_ptr, A.col_idx, A.values, r0, r1, p.lo, p.ext_len))
        self.buf = _DevBuf(16 * p.ext_len + 256)
        self.buf.tensor(16 * p.ext_len + 128, 1, "<i4").zero_()
        self.resolve = resolve
        self.epoch = 0

    def _flag_off(self, q):
        return 16 * self.plans[q].ext_len + 128

    def _ext(self, par):
        p = self.plans[self.rank]
        return self.buf.tensor(8 * par * p.ext_len, p.ext_len)

    def stage_input(self, x_local, epoch, s):
        from . import _native as N

        p = self.plans[self.rank]
        self._ext(epoch & 1)[p.own_offset : p.own_offset + (self.own[1] - self.own[0])].copy_(x_local)
        N.check(N.lib.sait_publish_epoch(C.c_void_p(self.buf.ptr + self._flag_off(self.rank)), int(epoch), s))

    def stage_spmv(self, y_local, epoch, s):
        from . import _native as N

        p = self.plans[self.rank]
        par = epoch & 1
        h = N.Halo()
        h.own_lo, h.own_hi, h.epoch = p.own[0] - p.lo, p.own[1] - p.lo, epoch
        for peer, g0, g1 in p.recv:
            pq = self.plans[peer]
            base = self.resolve(peer) + 8 * par * pq.ext_len
            flag = self.resolve(peer) + self._flag_off(peer)
            if g1 <= p.own[0]:
                h.lo_src, h.lo_shift, h.lo_flag = base, p.lo - pq.lo, flag
            else:
                h.hi_src, h.hi_shift, h.hi_flag = base, p.lo - pq.lo, flag
        x = self._ext(par)
        N.check(N.lib.sait_operator_apply_halo(self.op._h, x.data_ptr(), x.numel(), C.byref(h), y_local.data_ptr(),
                                               y_local.numel(), s))

    @classmethod
    def distributed(cls, A, rank: int, world: int, group=None, align: int = GROUP_ROWS):
        import torch.distributed as dist

        obj, mine, err = None, None, None
        try:
            obj = cls(A, rank, world, resolve=None, align=align)
            mine = obj.buf.handle()
        except Exception as exc:  # noqa: BLE001  (agreed on below)
            err = exc
        _agree(err, "PeerRowOperator", group, cleanup=obj)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        opened = {}
        try:
            for peer, _, _ in obj.plans[rank].recv:
                opened[peer] = _open_ipc(allh[peer])
        except Exception as exc:  # noqa: BLE001
            err = exc
        obj._opened = opened
        _agree(err, "PeerRowOperator", group, cleanup=obj)
        obj.resolve = lambda q: obj.buf.ptr if q == rank else opened[q]
        dist.barrier(group=group)
        return obj

    def close(self):
        from . import _native as N

        for p in getattr(self, "_opened", {}).values():
            N.lib.sait_ipc_close(C.c_void_p(p))
        self._opened = {}
        self.buf.free()
