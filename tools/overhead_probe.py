"""Per-call fixed overhead of xg.xigemm (host + launch + sync) at tiny sizes,
and the split between Python and the C-ABI call."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_06924_b200 as xg
from paper_2403_06924_b200 import api
for n in (256, 8192):
    a = xg.generate("student_t3", n, n, 1, 0.0, 1.0)
    b = xg.generate("student_t3", n, n, 2, 0.0, 1.0)
    cfg = xg.XigemmConfig(threshold=0.0154, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
    out = torch.empty((n, n), device="cuda")
    for _ in range(5):
        xg.xigemm(a, b, cfg=cfg, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 50
    e0.record()
    t0 = time.perf_counter()
    for _ in range(it):
        r = xg.xigemm(a, b, cfg=cfg, out=out)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / it * 1e6
    dev = e0.elapsed_time(e1) / it * 1e3
    stages = sum(v for k, v in r.timings.items() if k in ("quant", "xxmm", "reduce")) / 1e3
    # raw C-ABI call (no Python wrapper work besides ctypes)
    L = xg.lib()
    cfgc = cfg.c()
    rep = api.XgReport()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = (C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), None, C.c_float(1), C.c_float(0), n, n, n,
            C.byref(cfgc), 1, C.c_void_p(out.data_ptr()), C.byref(rep), None, s)
    t0 = time.perf_counter()
    for _ in range(it):
        L.xg_xigemm(*args)
    raw = (time.perf_counter() - t0) / it * 1e6
    print(f"n={n}: per call wall {wall:.1f} us, device-timed {dev:.1f} us, stage sum {stages:.1f} us, raw C call {raw:.1f} us")
