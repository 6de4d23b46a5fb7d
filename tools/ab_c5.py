"""C5-on-one-GPU timing of the package under ROOT (A/B of two trees on one box):
    python tools/ab_c5.py ROOT [M N K]"""
import os
import sys
import time

root = sys.argv[1]
sys.path.insert(0, root)
import torch  # noqa: E402

import paper_2403_06924_b200 as xg  # noqa: E402

m, n, k = (int(x) for x in (sys.argv[2:5] if len(sys.argv) >= 5 else (65536, 16384, 16384)))
a = xg.generate("normal", m, k, 1)
b = xg.generate("normal", k, n, 2)
out = torch.empty((m, n), dtype=torch.float32, device="cuda")
cfg = xg.XigemmConfig(threshold=0.0193, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
for _ in range(2):
    rep = xg.xigemm(a, b, cfg=cfg, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(4):
    rep = xg.xigemm(a, b, cfg=cfg, out=out)
e1.record()
torch.cuda.synchronize()
print(root, f"{m}x{n}x{k}", round(e0.elapsed_time(e1) / 4, 3), "ms", rep.timings, rep.density_a)
