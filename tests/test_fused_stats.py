"""Threshold statistics fused into the D_F GEMM's epilogue (EPI_DF_AVG /
EPI_DF_MIN, taken when the pair kernel runs and K >= 8192): the row / column
statistics of |D_F| (pipeline.cpp:215-247) must equal the oracle's bit for bit -
AvgRule through the verified-mean check over the epilogue's tree-ordered fp64
sums, MinRule exactly - on ragged shapes (partial row pairs, N not a multiple
of the 256-column tile or of the 16-column chunk), and the whole call must
equal the oracle, through the graph path as well as the stage-dump path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle_lib as ol  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2403_06924_b200 as xg  # noqa: E402
from test_gpu_parity import beq, cfg_from  # noqa: E402

SHAPES = [(300, 8192, 516), (513, 8192, 1028), (256, 9000, 260)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("scheme,pol", [(1, 0), (0, 1), (1, 1), (0, 0)], ids=["vw_avg", "pt_min", "vw_min", "pt_avg"])
def test_fused_stats_equal_oracle(oracle, shape, scheme, pol):
    m, k, n = shape
    a = ol.random_dense(m, k, m + 1, -3, 3)
    b = ol.random_dense(k, n, n + 2, -3, 3)
    a[m // 3, 5] = 25.0
    thr = 0.02 if pol == 0 else 2000.0
    c = ol.cfg(bits=8, threshold=thr, density_limit=0.9, scheme=scheme, policy=pol, rounding=1)
    rc, od = oracle.dump(a, b, c)
    assert rc == 0
    rep, d = xg.xigemm_dump(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), cfg_from(c))
    assert beq(d["d_f"], od["d_f"])
    assert beq(d["row_stat"], od["row_stat"]) and beq(d["col_stat"], od["col_stat"])
    assert beq(rep.result, od["result"])
    # the graph path (no dump: deferred exact means) on the second and third call
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    for _ in range(3):
        r = xg.xigemm(ta, tb, cfg=cfg_from(c), out=out)
        assert beq(out, od["result"])
        assert (r.density_a, r.density_b) == (rep.density_a, rep.density_b)


def test_fused_stats_widened_fallback():
    """XG_STATS_WIDEN=24 widens the verified interval so every AvgRule mean of
    the graph path takes the deferred exact fallback: the fused sums must still
    resolve to the reference's floats (the cases above in a subprocess; the
    hook is read once per process)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, XG_STATS_WIDEN="24")
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-x", "-k", "equal_oracle and avg",
                        "-p", "no:cacheprovider"], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.abspath(__file__)))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
