"""Quick device probe used during development: GEMM correctness + timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_06924_b200 as xg

def check(m, k, n):
    rng = np.random.default_rng(1)
    a = rng.integers(-127, 128, size=(m, k), dtype=np.int8)
    b = rng.integers(-127, 128, size=(k, n), dtype=np.int8)
    c = xg.gemm_i8(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    ref = (a.astype(np.int64) @ b.astype(np.int64)).astype(np.int32)
    bad = np.argwhere(c != ref)
    print(f"gemm {m}x{k}x{n}: mismatches={len(bad)}", bad[:5].tolist(), flush=True)
    if len(bad):
        i, j = bad[0]
        print("  got", c[i, j], "want", ref[i, j], flush=True)

print("device ok", xg.lib().xg_device_ok(), torch.cuda.get_device_name(0), flush=True)
for shp in [(128, 128, 256), (3, 3, 3), (256, 512, 512), (1000, 2000, 700)]:
    check(*shp)

def bench(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for n in (4096, 8192):
    a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    bT = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    ms = bench(lambda: xg.gemm_i8(a, bT))
    print(f"gemm_i8 {n}^3 (incl transpose+copy) {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TOPS", flush=True)
    A = xg.generate("student_t3", n, n, 1, 0, 1.0)
    B = xg.generate("student_t3", n, n, 2, 0, 1.0)
    for thr in (0.05, 0.1, 0.2):
        cfg = xg.XigemmConfig(threshold=thr, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
        rep = xg.xigemm(A, B, cfg=cfg)
        ms = bench(lambda: xg.xigemm(A, B, cfg=cfg), 5)
        print(f"xigemm {n}^3 t3 M={thr}: {ms:.3f} ms {2*n**3/ms/1e9:.1f} eff TOPS dens=({rep.density_a:.4f},{rep.density_b:.4f}) path={int(rep.path)} timings={rep.timings}", flush=True)
