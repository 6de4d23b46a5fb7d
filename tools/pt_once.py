"""C3 with the reference's default configuration (PerTensor, MinRule): stage
timings per call (profiling driver).  THR overrides the threshold M."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_06924_b200 as xg  # noqa: E402

n = int(os.environ.get("N", "8192"))
a = xg.generate("student_t3", n, n, 1)
b = xg.generate("student_t3", n, n, 2)
out = torch.empty((n, n), dtype=torch.float32, device="cuda")
cfg = xg.XigemmConfig(threshold=float(os.environ.get("THR", "0.01414")), scheme=xg.QuantScheme.PerTensor,
                      policy=xg.ReductionPolicy.MinRule)
for _ in range(int(os.environ.get("CALLS", "5"))):
    rep = xg.xigemm(a, b, cfg=cfg, out=out)
torch.cuda.synchronize()
print("density", rep.density_a, rep.density_b, int(rep.path), rep.timings)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = int(os.environ.get("STEPS", "20"))
e0.record()
for _ in range(steps):
    rep = xg.xigemm(a, b, cfg=cfg, out=out)
e1.record()
torch.cuda.synchronize()
st = rep.timings
print("per call %.1f us (events); stages quant %d df %d reduce %d comp %d us" % (
    e0.elapsed_time(e1) / steps * 1e3, st["quant"] // 1000, st["gemm_df"] // 1000, st["reduce"] // 1000,
    st["gemm_comp"] // 1000))
