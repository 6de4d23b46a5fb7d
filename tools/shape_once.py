"""A few xigemm calls at a given shape (M N K, data, threshold): profiling driver.
    M=16384 N=11008 K=4096 DIST_A=student_t3 DIST_B=normal THR=0.037 python tools/shape_once.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_06924_b200 as xg  # noqa: E402

m, n, k = (int(os.environ.get(x, "8192")) for x in ("M", "N", "K"))
a = xg.generate(os.environ.get("DIST_A", "student_t3"), m, k, 1)
b = xg.generate(os.environ.get("DIST_B", "student_t3"), k, n, 2)
out = torch.empty((m, n), dtype=torch.float32, device="cuda")
cfg = xg.XigemmConfig(threshold=float(os.environ.get("THR", "0.015")), scheme=xg.QuantScheme.VectorWise,
                      policy=xg.ReductionPolicy.AvgRule)
for _ in range(int(os.environ.get("CALLS", "3"))):
    rep = xg.xigemm(a, b, cfg=cfg, out=out)
torch.cuda.synchronize()
print("density", rep.density_a, rep.density_b, rep.timings)
