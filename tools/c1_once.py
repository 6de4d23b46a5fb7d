"""C1 (1024^3 uniform, VectorWise AvgRule ~5%) xigemm calls: timing with CUDA
events and the per-call host overhead (profiling driver)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_06924_b200 as xg  # noqa: E402

n = int(os.environ.get("N", "1024"))
a = xg.generate("uniform", n, n, 1, -1.0, 1.0)
b = xg.generate("uniform", n, n, 2, -1.0, 1.0)
out = torch.empty((n, n), dtype=torch.float32, device="cuda")
cfg = xg.XigemmConfig(threshold=0.112, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
for _ in range(5):
    rep = xg.xigemm(a, b, cfg=cfg, out=out)
torch.cuda.synchronize()
steps = int(os.environ.get("STEPS", "50"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(steps):
    rep = xg.xigemm(a, b, cfg=cfg, out=out)
e1.record()
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"C1 {n}^3: {e0.elapsed_time(e1) / steps * 1e3:.1f} us/call (events), {(t1 - t0) / steps * 1e6:.1f} us/call (wall), "
      f"density {rep.density_a:.4f}/{rep.density_b:.4f} path {int(rep.path)} kernel {rep.comp_kernel} "
      f"stages {rep.timings}")
