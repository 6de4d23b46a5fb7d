"""Row-sharded pipeline on one GPU: g shards run in one
process through the same staged C-ABI and protocol as the multi-GPU path,
with the collectives done in-process (LocalComm).  The concatenated rows must
equal the single-GPU xigemm bit for bit, and the report must be the global one."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle_lib as ol  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2403_06924_b200 as xg  # noqa: E402
from paper_2403_06924_b200 import sharded  # noqa: E402


def beq(x, y):
    x = x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
    y = y.cpu().numpy() if hasattr(y, "cpu") else np.asarray(y)
    return x.shape == y.shape and np.array_equal(x.view(np.uint32), y.view(np.uint32))


CFGS = [dict(bits=8, threshold=0.05, density_limit=0.5, scheme=1, policy=0, rounding=1),
        dict(bits=8, threshold=0.3, density_limit=0.5, scheme=0, policy=1, rounding=1),
        dict(bits=4, threshold=0.1, density_limit=0.3, scheme=1, policy=1, rounding=0),
        dict(bits=8, threshold=0.02, density_limit=1.0, scheme=0, policy=0, rounding=0)]


def _cfg(d):
    return xg.XigemmConfig(xg.QuantBits(d["bits"]), d["threshold"], d["density_limit"],
                           xg.QuantScheme(d["scheme"]), xg.ReductionPolicy(d["policy"]),
                           xg.RoundingMode(d["rounding"]))


@pytest.mark.parametrize("shape", [(300, 1024, 260), (97, 130, 70), (512, 2048, 1028)])
@pytest.mark.parametrize("g", [1, 2, 3, 4])
def test_sharded_equals_single(shape, g):
    m, k, n = shape
    a = torch.from_numpy(ol.random_dense(m, k, m + g, -4, 4)).cuda()
    b = torch.from_numpy(ol.random_dense(k, n, n + 1, -4, 4)).cuda()
    c = torch.from_numpy(ol.random_dense(m, n, 5, -1, 1)).cuda()
    a[m // 2, 3] = 41.0
    for d in CFGS:
        cfg = _cfg(d)
        ref = xg.xigemm(a, b, c, 1.25, -0.5, cfg)
        got = sharded.xigemm_sharded_local(a, b, c, 1.25, -0.5, cfg, nranks=g)
        assert beq(got.result, ref.result), (shape, g, d)
        assert (got.density_a, got.density_b, int(got.path), got.nnz_a, got.nnz_b) == \
               (ref.density_a, ref.density_b, int(ref.path), ref.nnz_a, ref.nnz_b)
        ref2 = xg.xigemm(a, b, None, 3.0, 0.0, cfg)
        got2 = sharded.xigemm_sharded_local(a, b, None, 3.0, 0.0, cfg, nranks=g)
        assert beq(got2.result, ref2.result)


def test_sharded_c3_like_vs_oracle():
    """Student-t data, AvgRule VectorWise at ~5% density (C3's settings), 4 shards."""
    m = k = n = 1024
    a = xg.generate("student_t3", m, k, 1, 0.0, 1.0)
    b = xg.generate("student_t3", k, n, 2, 0.0, 1.0)
    c = ol.cfg(threshold=0.05, density_limit=0.3, scheme=1, policy=0, rounding=1)
    rc, ref, orep = ol.oracle().xigemm(a.cpu().numpy(), b.cpu().numpy(), config=c)
    assert rc == 0
    got = sharded.xigemm_sharded_local(a, b, cfg=_cfg(dict(bits=8, threshold=0.05, density_limit=0.3, scheme=1,
                                                           policy=0, rounding=1)), nranks=4)
    assert beq(got.result, ref)
    assert (got.density_a, got.density_b, int(got.path)) == (orep.density_a, orep.density_b, orep.path)


def test_sharded_validation():
    a = torch.zeros((3, 8), device="cuda")
    b = torch.zeros((8, 4), device="cuda")
    with pytest.raises(xg.InvalidArgument):
        sharded.xigemm_sharded_local(a, b, nranks=4)  # fewer rows than ranks
    a[1, 2] = float("nan")
    with pytest.raises(xg.InvalidArgument):
        sharded.xigemm_sharded_local(a, b, nranks=2)  # NaN in one shard: every rank rejects


_WIDEN_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import oracle_lib as ol, paper_2403_06924_b200 as xg
from paper_2403_06924_b200 import sharded
cfg = xg.XigemmConfig(xg.QuantBits.Int8, 0.05, 0.5, xg.QuantScheme.VectorWise, xg.ReductionPolicy.AvgRule,
                      xg.RoundingMode.Nearest)
for seed in range(6):
    m, k, n = 200 + seed, 512, 12
    a = torch.from_numpy(ol.random_dense(m, k, seed + 1, -3, 3)).cuda()
    b = torch.from_numpy(ol.random_dense(k, n, seed + 2, -3, 3)).cuda()
    rc, ref, orep = ol.oracle().xigemm(a.cpu().numpy(), b.cpu().numpy(), config=ol.cfg(threshold=0.05,
                                       density_limit=0.5, scheme=1, policy=0, rounding=1))
    got = sharded.xigemm_sharded_local(a, b, cfg=cfg, nranks=3)
    assert np.array_equal(got.result.cpu().numpy().view(np.uint32), ref.view(np.uint32)), seed
# more flagged columns than the default 8-column exchange: XG_EAGAIN on every
# shard, the exchange grows to the reported count and the run is redone
grown = []
orig = sharded.Shard.grow_remote
def spy(self, needed):
    grown.append(needed)
    return orig(self, needed)
sharded.Shard.grow_remote = spy
m, k, n = 301, 512, 96
a = torch.from_numpy(ol.random_dense(m, k, 7, -3, 3)).cuda()
b = torch.from_numpy(ol.random_dense(k, n, 8, -3, 3)).cuda()
rc, ref, orep = ol.oracle().xigemm(a.cpu().numpy(), b.cpu().numpy(), config=ol.cfg(threshold=0.05,
                                   density_limit=0.5, scheme=1, policy=0, rounding=1))
got = sharded.xigemm_sharded_local(a, b, cfg=cfg, nranks=3)
assert np.array_equal(got.result.cpu().numpy().view(np.uint32), ref.view(np.uint32))
assert grown and max(grown) > 8, grown
print("ok", grown)
"""


def test_sharded_remote_exact_means_widened():
    """XG_STATS_WIDEN=40 flags every AvgRule mean (and widens the candidate interval to ~15%); column means whose kept set
    could change are recomputed from the all-gathered D_F columns in global row
    order (collective point 3).  Must still match the reference oracle."""
    here = os.path.dirname(os.path.abspath(__file__))
    code = _WIDEN_SCRIPT.format(root=os.path.dirname(here), tests=here)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, XG_STATS_WIDEN="40"),
                       capture_output=True, text=True)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


def test_sharded_nccl_graph_replay():
    """One-rank NCCL process group (torchrun): xigemm_sharded's eager first
    call and its CUDA-graph replays (stages + NCCL collectives captured) equal
    the single-GPU result bit for bit."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "tools", "shard_graph_check.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "equal single-GPU: True" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("g", [2, 3])
def test_sharded_csr_compensation(g):
    """The CUDA-core CSR compensation (forced) inside each shard: every rank's
    rows equal the single-GPU result (itself equal to the masked-dense launch)."""
    m, k, n = 700, 2052, 1028
    a = torch.from_numpy(ol.random_dense(m, k, m + 3, -4, 4)).cuda()
    b = torch.from_numpy(ol.random_dense(k, n, n + 5, -4, 4)).cuda()
    c = torch.from_numpy(ol.random_dense(m, n, 9, -1, 1)).cuda()
    cfg = _cfg(dict(bits=8, threshold=0.0202, density_limit=0.9, scheme=1, policy=0, rounding=1))
    saved = xg.comp_model()["force"]
    try:
        xg.comp_model(force=1)
        ref = xg.xigemm(a, b, c, 1.25, -0.5, cfg)
        xg.comp_model(force=2)
        got = sharded.xigemm_sharded_local(a, b, c, 1.25, -0.5, cfg, nranks=g)
    finally:
        xg.comp_model(force=saved)
    assert int(ref.path) == 0 and ref.comp_kernel == 0 and got.comp_kernel == 1
    assert beq(got.result, ref.result)
    assert (got.density_a, got.density_b, got.nnz_a, got.nnz_b) == (ref.density_a, ref.density_b, ref.nnz_a,
                                                                     ref.nnz_b)
