import time, sys, ctypes as C
sys.path.insert(0, '/root/repo')
import torch
import paper_2403_06924_b200 as xg
from paper_2403_06924_b200 import api
n = 256
a = xg.generate("student_t3", n, n, 1); b = xg.generate("student_t3", n, n, 2)
cfg = xg.XigemmConfig(threshold=0.0154, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
out = torch.empty((n, n), device="cuda")
def t(name, f, it=20000):
    f()
    t0 = time.perf_counter()
    for _ in range(it): f()
    print(f"{name:28s} {(time.perf_counter()-t0)/it*1e6:7.2f} us")
t("fast_dev x2", lambda: (api._fast_dev(a), api._fast_dev(b)))
t("check_out", lambda: api._check_out(out, n, n, a, b))
t("cfg.c()", lambda: cfg.c())
t("XgReport()", lambda: api.XgReport())
t("_s()", lambda: api._s())
t("_p x4", lambda: (api._p(a), api._p(b), api._p(None), api._p(out)))
t("lib()", lambda: api.lib())
rep = api.XgReport()
t("GemmReport build", lambda: api.GemmReport(out, rep.density_a, rep.density_b, api.GemmPath(rep.path),
     {"quant": int(rep.ns_quant), "xxmm": int(rep.ns_xxmm), "reduce": int(rep.ns_reduce), "package": int(rep.ns_package)},
     rep.nnz_a, rep.nnz_b, rep.stats_fallbacks, rep.comp_kernel))
t("xigemm full", lambda: xg.xigemm(a, b, cfg=cfg, out=out), 3000)
L = xg.lib(); cfgc = cfg.c(); r = api.XgReport(); s = api._s()
args = (C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), None, C.c_float(1), C.c_float(0), n, n, n, C.byref(cfgc), 1, C.c_void_p(out.data_ptr()), C.byref(r), None, s)
t("raw C xg_xigemm", lambda: L.xg_xigemm(*args), 3000)
