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
                  reduce_max=None):
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
        self.own = (r0, r1)
        self.ops, self.bufs = [], []
        for f, M in enumerate((ML, MU)):
            p = self.plans[f][rank]
            self.ops.append(DeviceOperator(local_block(M.row_ptr, M.col_idx, M.values, r0, r1, p.lo, p.ext_len)))
            self.bufs.append(_DevBuf(self._buf_bytes(f, rank)))
            self.bufs[f].tensor(self._flag_off(f, rank), 1, "<i4").zero_()
        self.resolve = resolve
        self.epoch = 0
        self.halo_bytes = 8 * sum(g1 - g0 for f in range(2) for _, g0, g1 in self.plans[f][rank].recv)

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

    def apply(self, r_local, z_local, stream=None) -> None:
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        self.epoch += 1
        self.stage_input(r_local, self.epoch, s)
        self.stage_lower(self.epoch, s)
        self.stage_upper(z_local, self.epoch, s)

    @classmethod
    def distributed(cls, ML, MU, rank: int, world: int, group=None, align: int = GROUP_ROWS):
        """Multi-process construction: the ranks swap IPC handles of their
        buffers (torch.distributed all_gather_object) and open their peers'."""
        import torch.distributed as dist

        obj, mine, err = None, None, None
        try:
            obj = cls(ML, MU, rank, world, resolve=None, align=align)
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
        dist.barrier(group=group)
        return obj

    def close(self):
        from . import _native as N

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
