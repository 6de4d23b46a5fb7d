"""One C3 xigemm at a given residual density with the compensation forced to the
CSR path (profiling driver: ncu captures its kernels)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_06924_b200 as xg  # noqa: E402

n = int(os.environ.get("N", "8192"))
thr = float(os.environ.get("THR", "0.0617"))  # ~0.1% density on the C3 inputs
force = int(os.environ.get("FORCE", "2"))
a = xg.generate("student_t3", n, n, 1)
b = xg.generate("student_t3", n, n, 2)
out = torch.empty((n, n), dtype=torch.float32, device="cuda")
cfg = xg.XigemmConfig(threshold=thr, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
xg.comp_model(force=force)
for _ in range(3):
    rep = xg.xigemm(a, b, cfg=cfg, out=out)
torch.cuda.synchronize()
print("density", rep.density_a, rep.density_b, "kernel", rep.comp_kernel, "comp_ms", rep.timings["gemm_comp"] * 1e-6)
