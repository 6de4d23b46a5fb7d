"""GEMM correctness + timing probe (both kernels: XG_GEMM_1CTA=1 forces 1-CTA)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_06924_b200 as xg

def check(m, k, n):
    rng = np.random.default_rng(m + k + n)
    a = rng.integers(-127, 128, size=(m, k), dtype=np.int8)
    b = rng.integers(-127, 128, size=(k, n), dtype=np.int8)
    c = xg.gemm_i8(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    ref = (a.astype(np.int64) @ b.astype(np.int64)).astype(np.int32)
    bad = np.argwhere(c != ref)
    print(f"gemm {m}x{k}x{n}: mismatches={len(bad)} {bad[:3].tolist()}", flush=True)

for shp in [(256, 128, 256), (256, 256, 512), (512, 1024, 768), (300, 200, 260), (1000, 4096, 700)]:
    check(*shp)
for n in (8192,):
    A = xg.generate("student_t3", n, n, 1, 0, 1.0)
    B = xg.generate("student_t3", n, n, 2, 0, 1.0)
    cfg = xg.XigemmConfig(threshold=0.01539926526059492, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
    for _ in range(3): rep = xg.xigemm(A, B, cfg=cfg)
    torch.cuda.synchronize()
    print({k: v / 1e3 for k, v in rep.timings.items()}, "us", flush=True)
import ctypes
