"""Compensation-kernel sweep on B200: xigemm with the sparse terms on the
tcgen05 masked-dense launch (force 1) and on the CUDA-core CSR SpMM (force 2),
and quantized_gemm_full_residual, at bisected residual densities on the C3
inputs (8192^3 Student-t(3), VectorWise, AvgRule).  Prints one JSON line per
density plus the device calibration (calibrate_eta)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2403_06924_b200 as xg  # noqa: E402


def timed(fn, steps=10, warmup=3):
    for _ in range(warmup):
        r = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, r


def main():
    n = int(os.environ.get("SWEEP_N", "8192"))
    m = int(os.environ.get("SWEEP_M", str(n)))
    k = int(os.environ.get("SWEEP_K", str(n)))
    kind = os.environ.get("SWEEP_DIST", "student_t3")
    dens = [float(x) for x in os.environ.get("SWEEP_DENS", "0.001,0.0025,0.005,0.01,0.02,0.05").split(",")]
    a = xg.generate(kind, m, k, 1)
    b = xg.generate(kind, k, n, 2)
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    s, p = xg.QuantScheme.VectorWise, xg.ReductionPolicy.AvgRule
    cfg0 = xg.XigemmConfig(threshold=0.3, scheme=s, policy=p)
    t_full, _ = timed(lambda: xg.quantized_gemm_full_residual(a, b, cfg0, out=out))
    for d in dens:
        thr = bench.find_threshold(xg, a, b, s, p, d, tol=0.15)
        cfg = xg.XigemmConfig(threshold=thr, scheme=s, policy=p)
        row = {"m": m, "n": n, "k": k, "dist": kind, "target": d, "threshold": thr}
        for name, f in (("dense", 1), ("csr", 2), ("auto", 0)):
            xg.comp_model(force=f)
            t, rep = timed(lambda: xg.xigemm(a, b, cfg=cfg, out=out))
            row[name + "_ms"] = t
            row[name + "_comp_ms"] = rep.timings["gemm_comp"] * 1e-6
            row[name + "_kernel"] = rep.comp_kernel
            row["density"] = max(rep.density_a, rep.density_b)
        row["full_residual_ms"] = t_full
        print(json.dumps(row), flush=True)
    xg.comp_model(force=0)
    for size in ((2048, 4096) if os.environ.get("SWEEP_CAL", "1") == "1" else ()):
        cal = xg.calibrate_eta(size, xg.QuantBits.Int8, 7)
        print(json.dumps({"calibrate_eta": size, "eta": cal.eta, "gemm_ops_per_s": cal.gemm_ops_per_s,
                          "spmm_macs_per_s": cal.spmm_macs_per_s}), flush=True)


if __name__ == "__main__":
    main()
