"""The real row-sharded kernels (xg_shard_*) in TWO processes on one GPU:
each process owns one rank's rows, and the couplings run through
torch.distributed (gloo; the exchange buffers are staged through host memory,
since NCCL needs one GPU per rank).  Every rank's rows must equal the
single-GPU xigemm bit for bit, with the global report.  The widened case
(XG_STATS_WIDEN) forces the point-3 exact-mean exchange past its default
capacity, so the XG_EAGAIN grow-and-rerun path runs across processes."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


class HostGlooComm:
    """sharded.DistComm over gloo with CUDA buffers staged through host memory."""

    def allreduce(self, ts, op):
        from paper_2403_06924_b200 import sharded
        o = {sharded.OP_MAX: dist.ReduceOp.MAX, sharded.OP_MIN: dist.ReduceOp.MIN,
             sharded.OP_SUM: dist.ReduceOp.SUM}[op]
        h = ts[0].cpu()
        dist.all_reduce(h, op=o)
        ts[0].copy_(h)

    def allgather(self, sends, recvs):
        h = sends[0].cpu()
        parts = [torch.empty_like(h) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, h)
        recvs[0].copy_(torch.cat(parts))


def _problem(case):
    import paper_2403_06924_b200 as xg
    m, k, n, thr = (515, 1024, 384, 0.05) if case == 0 else (301, 512, 96, 0.05)
    a = xg.generate("student_t3" if case == 0 else "uniform", m, k, 1, 0.0 if case == 0 else -3.0, 1.0 if case == 0 else 3.0)
    b = xg.generate("student_t3" if case == 0 else "uniform", k, n, 2, 0.0 if case == 0 else -3.0, 1.0 if case == 0 else 3.0)
    cfg = xg.XigemmConfig(threshold=thr, density_limit=0.5, scheme=xg.QuantScheme.VectorWise,
                          policy=xg.ReductionPolicy.AvgRule)
    return a, b, cfg


def _worker(rank, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from paper_2403_06924_b200 import sharded
    a, b, cfg = _problem(case)
    rows = sharded.split_rows(a.shape[0], 2)
    r0 = sum(rows[:rank])
    sh = sharded.Shard(a[r0:r0 + rows[rank]].contiguous(), b, None, 1.0, 0.0, rank, rows, cfg)
    grown = []
    while True:
        sharded.run_protocol([sh], HostGlooComm(), 2)
        try:
            rep = sh.finish()
            break
        except sharded.ShardRetry as e:
            grown.append(e.needed)
            sh.grow_remote(e.needed)
    q.put((rank, sh.out.cpu().numpy(), (rep.density_a, rep.density_b, rep.path, rep.nnz_a, rep.nnz_b), grown))
    sh.close()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", [0, 1])
def test_two_processes_equal_single_gpu(case, monkeypatch):
    import paper_2403_06924_b200 as xg
    if case == 1:
        monkeypatch.setenv("XG_STATS_WIDEN", "40")  # read by the spawned processes' library
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (o, rep, g)) for r, o, rep, g in (q.get(timeout=600) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b, cfg = _problem(case)
    ref = xg.xigemm(a, b, cfg=cfg)
    got = np.concatenate([res[0][0], res[1][0]])
    assert np.array_equal(got.view(np.uint32), ref.result.cpu().numpy().view(np.uint32))
    for r in range(2):
        assert res[r][1][:3] == (ref.density_a, ref.density_b, int(ref.path))
        assert res[r][1][3:] == (ref.nnz_a, ref.nnz_b)
    if case == 1:
        assert res[0][2] and res[0][2] == res[1][2] and max(res[0][2]) > 8
