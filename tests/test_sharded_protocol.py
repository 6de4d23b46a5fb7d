"""Host-side protocol of the row-sharded pipeline on CPU: two gloo ranks run
sharded.run_protocol over mock shards whose exchange buffers hold known
per-rank values; after every point each rank must hold the exact global
reduction (max / sum / min / all-gather in rank order), in the step order the
GPU shards expect."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2403_06924_b200 import sharded  # noqa: E402


class MockShard:
    def __init__(self, rank):
        self.rank, self.log, self.bufs = rank, [], {}
        r = rank + 1
        self.bufs[0] = [sharded.Exchange(torch.tensor([10 * r, 0, r % 2, 0], dtype=torch.int32), None,
                                         sharded.OP_MAX)]
        self.bufs[1] = [sharded.Exchange(torch.tensor([7 * r, 100 - r, 0, 0], dtype=torch.int32), None,
                                         sharded.OP_MAX)]
        self.bufs[2] = [sharded.Exchange(torch.tensor([0.5 * r, 1.25, 3.0 * r], dtype=torch.float64), None,
                                         sharded.OP_SUM)]
        send = torch.arange(4, dtype=torch.float32) + 10 * rank
        self.bufs[3] = [sharded.Exchange(send, torch.zeros(8, dtype=torch.float32), sharded.OP_ALLGATHER)]
        self.bufs[4] = [sharded.Exchange(torch.tensor([1000 + r], dtype=torch.int64), None, sharded.OP_SUM),
                        sharded.Exchange(torch.tensor([r * 3], dtype=torch.int32), None, sharded.OP_MAX)]
        for v in self.bufs.values():
            for e in v:
                if e.recv is None:
                    e.recv = e.send

    def step(self, p):
        self.log.append(("step", p))

    def exchanges(self, p):
        self.log.append(("exchange", p))
        return self.bufs.get(p, [])


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    sh = MockShard(rank)
    sharded.run_protocol([sh], sharded.DistComm(), 2)
    out = {p: [e.recv.tolist() for e in v] for p, v in sh.bufs.items()}
    q.put((rank, out, sh.log))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_protocol_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict((r, (o, lg)) for r, o, lg in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(60)
    assert res[0][0] == res[1][0]  # every rank holds the same reduced values
    out = res[0][0]
    assert out[0] == [[20, 0, 1, 0]]                 # MAX
    assert out[1] == [[14, 99, 0, 0]]                # MAX
    assert out[2] == [[1.5, 2.5, 9.0]]               # SUM
    assert out[3] == [[0, 1, 2, 3, 10, 11, 12, 13]]  # ALLGATHER in rank order
    assert out[4] == [[2003], [6]]                   # SUM int64, MAX
    want = [x for p in range(sharded.NSTEPS) for x in (("step", p), ("exchange", p))]
    assert res[0][1] == want and res[1][1] == want


def test_split_rows():
    assert sharded.split_rows(10, 3) == [4, 3, 3]
    assert sharded.split_rows(8192, 8) == [1024] * 8
    with pytest.raises(Exception):
        sharded.split_rows(2, 3)
