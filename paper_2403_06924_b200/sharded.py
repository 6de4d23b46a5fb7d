"""Row-sharded xigemm across ranks.

A and C are split by rows, B is replicated: ``broadcast_b`` ships it from one
rank with a single collective (NCCL over NVLink on a multi-GPU box).  Every
rank runs the staged C-ABI pipeline (``xg_shard_*`` in include/xigemm_c.h) on
its rows; between the stages the ranks perform the exact couplings the
reference's algorithm has (pipeline.cpp:50-111):

    point 0  max|A|                     (PerTensor scale)            MAX
    point 1  max|A|, max|RA|, NaN flag  (lambda_RA, MinRule scale)   MAX
    point 2  column statistics of D_F   (AvgRule sums / MinRule min) SUM / MIN
    point 3  D_F columns of the rare AvgRule means that need the exact
             sequential sum across ranks                            ALLGATHER
             (a fixed number of columns; a run that flags more raises
             ShardRetry on every rank and is rerun with a larger buffer)
    point 4  nnz(A'), retained max|A'|  (density, dispatch, scale)   SUM, MAX

All reductions are exact (max/min/integer sums) except the fp64 column sums,
whose rounding the verified-mean test covers for any order, so every rank's
rows equal the single-GPU result bit for bit.

Two communicators drive the same code:
  * ``DistComm``  - torch.distributed, one shard per process (``nccl`` on GPUs;
    ``gloo`` works for the host-side protocol tests);
  * ``LocalComm`` - all shards in one process on one GPU (the single-GPU
    simulation the parity tests use: g shards must reproduce xigemm exactly).
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import ShardRetry, XgReport, check, lib
from .api import comp_model, GemmPath, GemmReport, InvalidArgument, XigemmConfig, _dev, _p, _s

NSTEPS = 6
OP_MAX, OP_SUM, OP_MIN, OP_ALLGATHER = 0, 1, 2, 3
# uint32 payloads (non-negative float bit patterns, flags) travel as int32: all
# values are < 2^31, so signed max/min order them like the unsigned values.
_TYPESTR = {0: "<i4", 1: "<i8", 2: "<f8", 3: "<f4"}


class _DevView:
    """Zero-copy torch view of a device buffer owned by the C library."""

    def __init__(self, ptr: int, count: int, dtype: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": _TYPESTR[dtype],
                                         "data": (int(ptr), False), "version": 2}


def _view(ptr: int, count: int, dtype: int) -> torch.Tensor:
    return torch.as_tensor(_DevView(ptr, count, dtype), device="cuda")


class Exchange:
    def __init__(self, send: torch.Tensor, recv: torch.Tensor, op: int):
        self.send, self.recv, self.op = send, recv, op


class Shard:
    """One rank's rows of a row-sharded xigemm (owns the C handle)."""

    def __init__(self, a_rows, b, c_rows, alpha, beta, rank, rank_rows, cfg: XigemmConfig, reduce=True,
                 out=None):
        self.a, _ = _dev(a_rows, torch.float32)
        self.b, _ = _dev(b, torch.float32)
        self.c = None if c_rows is None else _dev(c_rows, torch.float32)[0]
        m, k = self.a.shape
        if self.b.shape[0] != k:
            raise InvalidArgument("xigemm: inner dimensions do not match")
        if rank_rows[rank] != m:
            raise InvalidArgument("xg_shard: row count of this rank does not match rank_rows")
        n = self.b.shape[1]
        if self.c is not None and tuple(self.c.shape) != (m, n):
            raise InvalidArgument("xigemm: C shape does not match the result")
        self.out = out if out is not None else torch.empty((m, n), dtype=torch.float32, device="cuda")
        self.nranks = len(rank_rows)
        self._ex = {}
        rr = (C.c_int * len(rank_rows))(*[int(r) for r in rank_rows])
        self._cfg = cfg.c()
        self.h = C.c_void_p()
        check(lib().xg_shard_create(_p(self.a), _p(self.b), _p(self.c), float(alpha), float(beta), int(rank),
                                    len(rank_rows), rr, k, n, C.byref(self._cfg), int(reduce), _p(self.out),
                                    C.byref(self.h)))

    def step(self, p: int) -> None:
        check(lib().xg_shard_step(self.h, p, _s()))

    def exchanges(self, p: int) -> list[Exchange]:
        """Collectives after step p (buffers are fixed for the handle's life: cached)."""
        if p not in self._ex:
            self._ex[p] = self._query(p)
        return self._ex[p]

    def _query(self, p: int) -> list[Exchange]:
        res, i = [], 0
        while True:
            send, recv = C.c_void_p(), C.c_void_p()
            cnt, dt, op = C.c_int64(), C.c_int(), C.c_int()
            check(lib().xg_shard_exchange(self.h, p, i, C.byref(send), C.byref(recv), C.byref(cnt),
                                          C.byref(dt), C.byref(op)))
            if cnt.value == 0:
                return res
            sv = _view(send.value, cnt.value, dt.value)
            rv = _view(recv.value, cnt.value * self.nranks, dt.value) if op.value == OP_ALLGATHER else sv
            res.append(Exchange(sv, rv, op.value))
            i += 1

    def finish(self) -> XgReport:
        """Synchronises and returns the global report; the handle (and its
        workspace) stays valid for the next run of the same problem.  Raises
        ShardRetry (on every rank alike) when the run flagged more exact column
        means than the point-3 exchange holds: grow_remote(), then rerun."""
        rep = XgReport()
        try:
            check(lib().xg_shard_finish(self.h, C.byref(rep), _s()))
        except ShardRetry as e:
            e.needed = int(lib().xg_shard_remote_needed(self.h))
            raise
        return rep

    def grow_remote(self, needed: int) -> None:
        """Point-3 exchange buffer for `needed` columns (new buffers: re-queried)."""
        check(lib().xg_shard_set_remote_cap(self.h, int(needed)))
        self._ex.clear()
        self._graph = None

    def close(self):
        if self.h:
            lib().xg_shard_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class LocalComm:
    """All shards in this process (one GPU): collectives are local reductions."""

    def allreduce(self, ts: list[torch.Tensor], op: int) -> None:
        st = torch.stack(ts)
        r = st.amax(0) if op == OP_MAX else st.amin(0) if op == OP_MIN else st.sum(0)
        for t in ts:
            t.copy_(r)

    def allgather(self, sends: list[torch.Tensor], recvs: list[torch.Tensor]) -> None:
        cat = torch.cat(sends)
        for r in recvs:
            r.copy_(cat)


class DistComm:
    """torch.distributed, one shard per process (nccl on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def allreduce(self, ts: list[torch.Tensor], op: int) -> None:
        d = self.dist
        o = {OP_MAX: d.ReduceOp.MAX, OP_MIN: d.ReduceOp.MIN, OP_SUM: d.ReduceOp.SUM}[op]
        d.all_reduce(ts[0], op=o, group=self.group)

    def allgather(self, sends: list[torch.Tensor], recvs: list[torch.Tensor]) -> None:
        self.dist.all_gather_into_tensor(recvs[0], sends[0], group=self.group)


def run_protocol(shards: list, comm, nranks: int) -> None:
    """Steps 0..5 with the point-p collectives after step p, in lockstep over
    the shards this process holds (one per process with DistComm).  Works for
    any object with step(p) / exchanges(p) (the CPU protocol tests use mocks)."""
    for p in range(NSTEPS):
        for sh in shards:
            sh.step(p)
        per = [sh.exchanges(p) for sh in shards]
        for i in range(len(per[0])):
            ex = [x[i] for x in per]
            if ex[0].op == OP_ALLGATHER:
                comm.allgather([e.send for e in ex], [e.recv for e in ex])
            else:
                comm.allreduce([e.send for e in ex], ex[0].op)


def _report(rep: XgReport, result) -> GemmReport:
    return GemmReport(result, rep.density_a, rep.density_b, GemmPath(rep.path), {}, rep.nnz_a, rep.nnz_b,
                      rep.stats_fallbacks, rep.comp_kernel)  # comp_kernel: this rank's compensation kernel


_replayed_launches = 0


def launch_count(reset: bool = False) -> int:
    """This library's kernel launches (xg_launch_count) plus those replayed inside
    the shards' captured CUDA graphs (which the library does not see)."""
    global _replayed_launches
    n = int(lib().xg_launch_count(1 if reset else 0)) + _replayed_launches
    if reset:
        _replayed_launches = 0
    return n


def split_rows(m: int, nranks: int) -> list[int]:
    """Balanced contiguous row blocks (the first m % nranks ranks get one more)."""
    if m < nranks:
        raise InvalidArgument("xg_shard: fewer rows than ranks")
    q, r = divmod(m, nranks)
    return [q + (1 if i < r else 0) for i in range(nranks)]


def xigemm_sharded_local(a, b, c=None, alpha: float = 1.0, beta: float = 0.0,
                         cfg: XigemmConfig | None = None, nranks: int = 2, reduce: bool = True) -> GemmReport:
    """Single-process simulation of the nranks-way row-sharded pipeline on the
    current GPU (LocalComm).  Must equal xigemm(a, b, c, ...) bit for bit."""
    cfg = cfg or XigemmConfig()
    x, _ = _dev(a, torch.float32)
    y, _ = _dev(b, torch.float32)
    cc = None if c is None else _dev(c, torch.float32)[0]
    rows = split_rows(x.shape[0], nranks)
    out = torch.empty((x.shape[0], y.shape[1]), dtype=torch.float32, device="cuda")
    shards, r0 = [], 0
    for r, m in enumerate(rows):
        shards.append(Shard(x[r0:r0 + m], y, None if cc is None else cc[r0:r0 + m], alpha, beta, r, rows, cfg,
                            reduce, out[r0:r0 + m]))
        r0 += m
    try:
        while True:
            run_protocol(shards, LocalComm(), nranks)
            try:
                reps = [sh.finish() for sh in shards]
                break
            except ShardRetry as e:  # rare: more exact column means than the exchange holds
                for sh in shards:
                    sh.grow_remote(e.needed)
    finally:
        for sh in shards:
            sh.close()
    return _report(reps[0], out)


def broadcast_b(b: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Replicates B from rank `src` with one collective (ncclBroadcast)."""
    import torch.distributed as dist
    dist.broadcast(b, src=src, group=group)
    return b


_SHARD_CACHE: dict = {}
_SHARD_CACHE_MAX = 2


def _cached_shard(key, make):
    """Reuses the handle (persistent workspace, no per-call allocation) of a
    repeated call; at most _SHARD_CACHE_MAX problems are kept."""
    sh = _SHARD_CACHE.pop(key, None)
    if sh is None:
        while len(_SHARD_CACHE) >= _SHARD_CACHE_MAX:
            _SHARD_CACHE.pop(next(iter(_SHARD_CACHE))).close()
        sh = make()
    _SHARD_CACHE[key] = sh
    return sh


def xigemm_sharded(a_rows, b, c_rows=None, alpha: float = 1.0, beta: float = 0.0,
                   cfg: XigemmConfig | None = None, *, group=None, reduce: bool = True, out=None,
                   rank_rows: list[int] | None = None, graph: bool = True) -> GemmReport:
    """This rank's rows of the row-sharded xigemm (torch.distributed must be
    initialised; B must already be identical on every rank, see broadcast_b).
    rank_rows (every rank's row count) is all-gathered when not given.  From the
    second call of the same problem on, the stages and collectives replay as one
    CUDA graph (graph=False disables).  Returns the global report with this
    rank's result rows."""
    import torch.distributed as dist
    cfg = cfg or XigemmConfig()
    x, _ = _dev(a_rows, torch.float32)
    y, _ = _dev(b, torch.float32)
    cc = None if c_rows is None else _dev(c_rows, torch.float32)[0]
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if rank_rows is None:
        mine = torch.tensor([x.shape[0]], dtype=torch.int64, device="cuda")
        allm = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allm, mine, group=group)
        rank_rows = [int(t) for t in torch.cat(allm).tolist()]
    if out is not None and (not isinstance(out, torch.Tensor) or not out.is_cuda or out.dtype != torch.float32
                            or tuple(out.shape) != (x.shape[0], y.shape[1]) or not out.is_contiguous()):
        raise InvalidArgument("xigemm: out must be a contiguous float32 CUDA tensor of the result's shape")
    c = cfg.c()
    # out=None: the cached shard's own result buffer is reused (and returned), so
    # a repeated call hits the cache (and its CUDA graph) instead of a new handle
    key = (x.data_ptr(), tuple(x.shape), y.data_ptr(), tuple(y.shape), 0 if cc is None else cc.data_ptr(),
           None if out is None else out.data_ptr(), float(alpha), float(beta), bool(reduce), rank, tuple(rank_rows),
           (c.bits, c.threshold, c.density_limit, c.scheme, c.policy, c.rounding), id(group),
           tuple(comp_model().values()))  # the handle holds the compensation cost model of its creation
    sh = _cached_shard(key, lambda: Shard(x, y, cc, alpha, beta, rank, rank_rows, cfg, reduce, out))
    runs = getattr(sh, "_runs", 0)
    if graph and runs >= 1 and getattr(sh, "_graph", None) is None:
        # second call of the same problem: capture the six stages and their NCCL
        # collectives once, replay from then on (one launch per call)
        g = torch.cuda.CUDAGraph()
        n0 = lib().xg_launch_count(0)
        with torch.cuda.graph(g):
            run_protocol([sh], DistComm(group), world)
        sh._graph_launches = int(lib().xg_launch_count(0) - n0)  # kernels inside the captured graph
        sh._graph = g
    if getattr(sh, "_graph", None) is not None:
        sh._graph.replay()
        global _replayed_launches
        _replayed_launches += sh._graph_launches
    else:
        run_protocol([sh], DistComm(group), world)
    sh._runs = runs + 1
    while True:
        try:
            return _report(sh.finish(), sh.out)
        except ShardRetry as e:  # every rank raises alike: grow the exchange, rerun eagerly
            sh.grow_remote(e.needed)
            run_protocol([sh], DistComm(group), world)
