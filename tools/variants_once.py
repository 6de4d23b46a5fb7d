"""C3 xigemm under non-default configurations (Floor rounding, PerTensor
AvgRule, MinRule VectorWise): per-stage times and the launch path (profiling
driver for the generic kernels)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2403_06924_b200 as xg  # noqa: E402

n = int(os.environ.get("N", "8192"))
a = xg.generate("student_t3", n, n, 1)
b = xg.generate("student_t3", n, n, 2)
out = torch.empty((n, n), dtype=torch.float32, device="cuda")
for name, scheme, policy, rnd in (("VW Avg Nearest", 1, 0, 1), ("VW Avg Floor", 1, 0, 0), ("PT Avg Nearest", 0, 0, 1),
                                  ("VW Min Nearest", 1, 1, 1)):
    s, p = xg.QuantScheme(scheme), xg.ReductionPolicy(policy)
    thr = bench.find_threshold(xg, a, b, s, p, 0.05)
    cfg = xg.XigemmConfig(threshold=thr, scheme=s, policy=p, rounding=xg.RoundingMode(rnd))
    for _ in range(3):
        rep = xg.xigemm(a, b, cfg=cfg, out=out)
    t, rep = bench.time_calls(xg, torch, a, b, cfg, out, 10, 2)
    print(f"{name}: {t * 1e3:.3f} ms  density {max(rep.density_a, rep.density_b):.4f} path {int(rep.path)} "
          f"{rep.timings}", flush=True)
