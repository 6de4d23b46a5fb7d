"""Host-buffer e2e probe: host copy bandwidth and the pageable xg_xigemm_host call at C3."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2403_06924_b200 as xg
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
x = np.random.rand(64 << 20).astype(np.float32); y = np.empty_like(x)
t0=time.perf_counter(); 
for _ in range(5): np.copyto(y, x)
print("numpy copy GB/s", 5*x.nbytes/(time.perf_counter()-t0)/1e9)
m=n=k=8192
a = xg.generate("student_t3", m, k, 1); b = xg.generate("student_t3", k, n, 2)
cfg = xg.XigemmConfig(threshold=0.015, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
an, bn = a.cpu().numpy(), b.cpu().numpy(); on = np.empty((m, n), np.float32)
for _ in range(2): xg.xigemm_host(an, bn, cfg=cfg, out=on)
t0=time.perf_counter()
for _ in range(5): xg.xigemm_host(an, bn, cfg=cfg, out=on)
print(os.environ.get("XG_COPY_THREADS"), "pageable ms", (time.perf_counter()-t0)/5*1e3)
