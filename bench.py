"""Benchmark of the compensated INT8 GEMM (arXiv 2403.06924 "xigemm") on B200.

One step = one full xigemm() over one synthetic batch: quantize A and B,
tcgen05 INT8 GEMM, |D_F| statistics, residual quantisation + threshold
selection, compensation with the fused epilogue.  Metric (BASELINE.json):
effective TFLOP/s = 2MNK / t, plus the relative error against an FP64 GEMM.

Workload (headline): C3 of BASELINE.json - M=N=K=8192, Student-t(3) FP32
inputs, INT8 vector-wise quantisation, AvgRule, threshold M bisected for ~5%
residual density (s = 0.3, sparse path).  Inputs (256 MiB each) exceed the
126 MB L2, so no explicit flush is needed between steps.  The same JSON line
carries every other configuration of BASELINE.json (C1, C2 at 1/5/10%, C4, C5
on one GPU, C3 under the reference's default PerTensor/MinRule), each against
the roofline of SURVEY.md section 8(d).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU (torchrun, --gpus N > 1): the row-sharded pipeline (weak scaling:
M rows of A and C per GPU, B broadcast from rank 0 by NCCL every step, exact
all-reduce couplings between the stages; paper_2403_06924_b200/sharded.py).
--replicas runs N independent full problems instead.

The reference arm (--impl reference) never loads this repository's CUDA
library: inputs come from numpy, and the reference's own xigemm (oracle/_ref,
compiled from the reference sources) is timed on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M_DEFAULT = N_DEFAULT = K_DEFAULT = 8192
TARGET_DENSITY = 0.05
# M giving ~5% density on the C3 inputs (bisected on the device generator's
# Student-t(3) data: density 4.69%); the reference arm, which must not load the
# CUDA library, uses it for its numpy-generated inputs of the same distribution
C3_THRESHOLD = 0.01539926526059492
P_I8_SPEC = 4.5e15   # B200 dense INT8 op/s
BW_SPEC = 8.0e12     # HBM3e B/s (north star "~8 TB/s")
METRIC = "effective TFLOP/s (2MNK/t) of compensated GEMM"


def _dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or "MASTER_ADDR" in os.environ:
        import torch
        import torch.distributed as dist
        backend = "nccl" if os.environ.get("XG_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(backend)
    return world, rank, local


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop = [], 0, threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        s = sorted(self.samples)
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(s)}


def _peaks_file():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6448.4)) * 1e9, float(d.get("bf16_tflops", 1675.7)) * 1e12, "measured"
    except OSError:
        return 6.4484e12, 1.6757e12, "fallback (B200_PROFILING.md figures)"


# ---------------------------------------------------------------- roofline --
def b_alg(m, n, k, nnz_a, nnz_b):
    """Algorithmic bytes of one single-GPU call:
    A, B fp32 read twice (phases Q and R), Aq/Bq/RAq/RBq written and read,
    D_F written and read, C written, CSR(A') / CSR(B'^T) col_idx + int8 value
    written and read, row pointers written and read."""
    return 12 * (m * k + k * n) + 12 * m * n + 10 * (nnz_a + nnz_b) + 8 * (m + n + 2)


def roofline(m, n, k, nnz_a, nnz_b, t_s, p_i8=P_I8_SPEC, bw=BW_SPEC, p_simt=None):
    """T_roof = 2MNK/P_i8 + B_alg/BW (summed: the phases are data-dependent);
    frac = T_roof / t = achieved effective TFLOP/s / roofline effective TFLOP/s.
    With p_simt, the 3-term model adds the SpMM MACs (nnzA*N + nnzB*M) at the
    measured SIMT integer MAC rate."""
    ops = 2.0 * m * n * k
    ba = b_alg(m, n, k, nnz_a, nnz_b)
    t_tc, t_hbm = ops / p_i8, ba / bw
    t_roof = t_tc + t_hbm
    r = {"t_roof_us": t_roof * 1e6, "tensor_us": t_tc * 1e6, "hbm_us": t_hbm * 1e6, "b_alg_bytes": ba,
         "peak": ops / t_roof / 1e12, "achieved": ops / t_s / 1e12, "frac": t_roof / t_s}
    if p_simt:
        t3 = t_roof + (float(nnz_a) * n + float(nnz_b) * m) / p_simt
        r["three_term"] = {"simt_macs": float(nnz_a) * n + float(nnz_b) * m, "t_roof_us": t3 * 1e6,
                           "frac": t3 / t_s}
    return r


def measure_peaks(L):
    """INT8 tensor ceiling from the repo's own tcgen05 GEMM with TMA loads and
    epilogue switched off (MMA issue only, 8192^3), SIMT integer MAC rates
    (IDP4A, IMAD) from probe kernels; HBM from MEASURED_PEAKS.json."""
    hbm, bf16, src = _peaks_file()
    out = {"hbm_Bps": hbm, "hbm_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
           "bf16_flops": bf16}
    try:
        L.xg_debug_gemm_df.restype = C.c_double
        L.xg_debug_gemm_df.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        ms = L.xg_debug_gemm_df(8192, 8192, 8192, 1 | 2, 20)
        out["int8_ops"] = 2.0 * 8192 ** 3 / (ms * 1e-3) if ms > 0 else None
        out["int8_source"] = "tcgen05 kind::i8 pair GEMM, MMA issue only (debug flags: no TMA, no epilogue), 8192^3"
    except AttributeError:
        out["int8_ops"] = None
    try:
        L.xg_debug_simt_rate.restype = C.c_double
        L.xg_debug_simt_rate.argtypes = [C.c_int, C.c_int]
        out["idp4a_macs"] = L.xg_debug_simt_rate(0, 4096)
        out["imad_macs"] = L.xg_debug_simt_rate(1, 4096)
    except AttributeError:
        out["idp4a_macs"] = out["imad_macs"] = None
    if not out.get("int8_ops"):
        out["int8_ops"], out["int8_source"] = 2.0 * bf16, "2 x MEASURED_PEAKS bf16_tflops (proxy)"
    return out


# --------------------------------------------------------------- workloads --
def find_threshold(xg, a, b, scheme, policy, target=TARGET_DENSITY, tol=0.1):
    """Bisects M (log scale) so max(density_a, density_b) is within tol*target.
    MinRule thresholds scale with the operand sizes (sparse.cpp:49-55: M * lambda'
    * min|D_F| / K), so the range reaches far above AvgRule's (~1e-2)."""
    lo, hi = 1e-5, 1e7
    best = None
    for _ in range(40):
        mid = (lo * hi) ** 0.5
        rep = xg.xigemm(a, b, cfg=xg.XigemmConfig(threshold=mid, scheme=scheme, policy=policy))
        d = max(rep.density_a, rep.density_b)
        if best is None or abs(d - target) < abs(best[1] - target):
            best = (mid, d)
        if abs(d - target) <= tol * target:
            break
        if d > target:
            lo = mid
        else:
            hi = mid
    return best[0]


CONFIGS = [
    # name, m, n, k, A data, B data, scheme, policy, target density
    ("C1 1024^3 uniform VectorWise AvgRule 5%", 1024, 1024, 1024, ("uniform", -1.0, 1.0), ("uniform", -1.0, 1.0),
     1, 0, 0.05),
    ("C2 4096^3 normal VectorWise AvgRule 1%", 4096, 4096, 4096, ("normal", 0.0, 1.0), ("normal", 0.0, 1.0), 1, 0,
     0.01),
    ("C2 4096^3 normal VectorWise AvgRule 5%", 4096, 4096, 4096, ("normal", 0.0, 1.0), ("normal", 0.0, 1.0), 1, 0,
     0.05),
    ("C2 4096^3 normal VectorWise AvgRule 10%", 4096, 4096, 4096, ("normal", 0.0, 1.0), ("normal", 0.0, 1.0), 1, 0,
     0.10),
    # PerTensor on Student-t(3): most of Aq / Bq quantise to 0, so every row and
    # column of D_F holds an exact 0, min|D_F| = 0 and MinRule keeps every entry
    # whatever M (tools/minrule_probe.py): the reference's defaults run its
    # DenseResidual branch here (density 1.0), the bisection cannot reach 5%
    ("C3 8192^3 Student-t(3) PerTensor MinRule (reference defaults; density 1.0, DenseResidual)", 8192, 8192, 8192,
     ("student_t3", 0.0, 1.0), ("student_t3", 0.0, 1.0), 0, 1, 0.05),
    ("C4 16384x11008x4096 A Student-t(3) B normal VectorWise AvgRule 5%", 16384, 11008, 4096,
     ("student_t3", 0.0, 1.0), ("normal", 0.0, 1.0), 1, 0, 0.05),
    ("C5 65536x16384x16384 normal VectorWise AvgRule 5% (one GPU)", 65536, 16384, 16384, ("normal", 0.0, 1.0),
     ("normal", 0.0, 1.0), 1, 0, 0.05),
]


def time_calls(xg, torch, a, b, cfg, out, steps, warmup):
    for _ in range(warmup):
        rep = xg.xigemm(a, b, cfg=cfg, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        rep = xg.xigemm(a, b, cfg=cfg, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e-3, rep


def run_configs(xg, torch, peaks, steps, only=None):
    res = []
    for name, m, n, k, da, db, scheme, policy, target in CONFIGS:
        if only and not any(o in name for o in only):
            continue
        try:
            a = xg.generate(da[0], m, k, 1, da[1], da[2])
            b = xg.generate(db[0], k, n, 2, db[1], db[2])
            s, p = xg.QuantScheme(scheme), xg.ReductionPolicy(policy)
            thr = find_threshold(xg, a, b, s, p, target)
            cfg = xg.XigemmConfig(threshold=thr, scheme=s, policy=p)
            out = torch.empty((m, n), dtype=torch.float32, device="cuda")
            big = m * n * k > 2 ** 36
            t, rep = time_calls(xg, torch, a, b, cfg, out, max(3, steps // (4 if big else 1)), 3)
            rf = roofline(m, n, k, rep.nnz_a, rep.nnz_b, t)
            rm = roofline(m, n, k, rep.nnz_a, rep.nnz_b, t, peaks["int8_ops"], peaks["hbm_Bps"],
                          peaks.get("idp4a_macs"))
            res.append({"config": name, "m": m, "n": n, "k": k, "threshold_M": thr,
                        "density_a": rep.density_a, "density_b": rep.density_b, "path": int(rep.path),
                        "ms": t * 1e3, "tflops": 2.0 * m * n * k / t / 1e12,
                        "t_roof_us": rf["t_roof_us"], "frac": rf["frac"],
                        "frac_measured_peaks": rm["frac"],
                        "frac_three_term": rm.get("three_term", {}).get("frac"),
                        "gemm_df_ms": rep.timings["gemm_df"] * 1e-6, "gemm_comp_ms": rep.timings["gemm_comp"] * 1e-6})
            del a, b, out
            torch.cuda.empty_cache()
        except Exception as ex:  # noqa: BLE001
            res.append({"config": name, "error": str(ex)[:300]})
    return res


# ------------------------------------------------------------- CPU baseline --
def _reference_lib():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol
    r = ol.reference()
    if r is not None:
        return ol, r, "reference"
    return ol, ol.oracle(), "port"


def slab_fit(ol, r, a_rows, b, thr, scheme, policy, sizes=(16, 48), threads=1, reps=1):
    """The reference's xigemm on row slabs of A against the full B (on `threads`
    host threads at once, each its own slab): t(rows) = t_B + rows * t_row,
    where t_B is the per-call O(KN) B-side work and t_row the per-row work.
    Returns (t_B, t_row, densities of the largest slab, wall seconds)."""
    import numpy as np
    cfg = ol.cfg(threshold=thr, density_limit=0.3, scheme=scheme, policy=policy, rounding=1)
    k, n = b.shape
    times, dens = {}, None
    w0 = time.perf_counter()
    for rows in sizes:
        slabs = [np.ascontiguousarray(a_rows[(t * rows) % max(1, a_rows.shape[0] - rows):][:rows])
                 for t in range(threads)]
        outs = [None] * threads

        def work(t):
            outs[t] = r.xigemm(slabs[t], b, config=cfg)

        best = None
        for _ in range(reps):
            t0 = time.perf_counter()
            ths = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
            for th in ths:
                th.start()
            for th in ths:
                th.join()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        times[rows] = best
        dens = (outs[0][2].density_a, outs[0][2].density_b)
    r1, r2 = sizes
    t_row = max(1e-9, (times[r2] - times[r1]) / (r2 - r1))
    t_b = max(0.0, times[r1] - r1 * t_row)
    return t_b, t_row, dens, time.perf_counter() - w0


def cpu_baseline_run(jobs):
    """1-core reference timings (bench.py cpu_baseline): C1 and C2 on the full
    problem with the GPU arm's inputs and thresholds (best of 3 / once; the
    outputs are compared bit for bit with the GPU's), C3 by the two-slab fit."""
    import numpy as np
    ol, r, kind = _reference_lib()
    res = {"kind": kind, "cores": 1}
    for job in jobs:
        name, a, b, thr, scheme, policy, gpu_out = job["name"], job["a"], job["b"], job["thr"], job["scheme"], \
            job["policy"], job.get("gpu_out")
        m, k = a.shape
        n = b.shape[1]
        cfg = ol.cfg(threshold=thr, density_limit=0.3, scheme=scheme, policy=policy, rounding=1)
        if job["mode"] == "full":
            best = None
            for _ in range(job.get("reps", 1)):
                t0 = time.perf_counter()
                rc, out, rep = r.xigemm(a, b, config=cfg)
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            d = {"mode": f"full problem, best of {job.get('reps', 1)}", "seconds": best,
                 "tflops": 2.0 * m * n * k / best / 1e12, "density_a": rep.density_a, "density_b": rep.density_b}
            if gpu_out is not None:
                d["bit_equal_to_gpu"] = bool(np.array_equal(out.view(np.uint32), gpu_out.view(np.uint32)))
        else:
            t_b, t_row, dens, wall = slab_fit(ol, r, a, b, thr, scheme, policy)
            t_full = t_b + m * t_row
            d = {"mode": "two-slab fit: xigemm_ref on 16- and 48-row slabs of A with the full B, "
                         "t = t_B + M * t_row (estimate)", "t_B_s": t_b, "t_row_s": t_row, "seconds": t_full,
                 "tflops": 2.0 * m * n * k / t_full / 1e12, "density_a_slab": dens[0],
                 "density_b_slab": dens[1], "sample_wall_s": wall}
        res[name] = d
    return res


def run_reference(args, world, rank):
    """--impl reference: the reference's own xigemm (oracle/_ref) on this box's
    host cores, on the C3 workload, without this repository's CUDA library.
    Inputs: numpy Student-t(3) of the same shape and distribution; threshold
    C3_THRESHOLD (or --threshold).  Each step runs T concurrent slabs (one per
    host thread, alternating 16- and 48-row slabs of A against the full B);
    the fit t(rows) = t_B + rows*t_row over the steps gives the time of the
    whole problem with the row work spread over the T threads:
    t = t_B + M*t_row/T (the B-side work of the reference is serial)."""
    import numpy as np
    if world > 1 and rank != 0:
        return
    ol, r, kind = _reference_lib()
    m, n, k = args.m, args.n, args.k
    threads = min(os.cpu_count() or 1, 64)
    try:
        import psutil
        threads = max(1, min(threads, int(psutil.virtual_memory().available / 2.5e9)))
    except Exception:  # noqa: BLE001
        pass
    thr = args.threshold if args.threshold is not None else C3_THRESHOLD
    rng = np.random.default_rng(1)
    small, big = (2, 6) if args.ref_rows_set and args.ref_rows <= 4 else (16, 48)
    nrows = big * threads + big

    def t3(rows, cols):
        z = rng.standard_normal((rows, cols), dtype=np.float32)
        chi = (rng.standard_normal((3, rows, cols), dtype=np.float32) ** 2).sum(0) / np.float32(3.0)
        return (z / np.sqrt(chi)).astype(np.float32)

    a = t3(min(m, nrows), k)
    b = t3(k, n)
    cfg = ol.cfg(threshold=thr, density_limit=0.3, scheme=1, policy=0, rounding=1)
    nsteps = max(1, args.steps if args.ref_steps is None else args.ref_steps)
    samples = {small: [], big: []}
    dens = None
    for i in range(nsteps):
        rows = small if i % 2 == 0 else big
        slabs = [np.ascontiguousarray(a[(t * rows) % max(1, a.shape[0] - rows):][:rows]) for t in range(threads)]
        outs = [None] * threads

        def work(t):
            outs[t] = r.xigemm(slabs[t], b, config=cfg)

        t0 = time.perf_counter()
        ths = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        samples[rows].append(time.perf_counter() - t0)
        if rows == big or dens is None:
            dens = (outs[0][2].density_a, outs[0][2].density_b)
    ts = {s: sorted(v)[len(v) // 2] for s, v in samples.items() if v}
    if len(ts) == 2:
        t_row = max(1e-9, (ts[big] - ts[small]) / (big - small))
        t_b = max(0.0, ts[small] - small * t_row)
    else:  # one step only: no fit, the slab's B-side share is charged to its rows
        t_b, t_row = 0.0, ts[small] / small
    t_full = t_b + m * t_row / threads
    value = 2.0 * m * n * k / t_full / 1e12
    sample = (f"{threads} host threads, each xigemm_ref on its own {small}- or {big}-row slab of A against the "
              f"full {k}x{n} B per step (alternating); fit t(rows) = t_B + rows*t_row: t_B = {t_b:.2f} s, "
              f"t_row = {t_row * 1e3:.1f} ms; C3 time = t_B + M*t_row/threads = {t_full:.1f} s")
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": nsteps,
        "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8/fp64 (reference CPU)",
        "data": "synthetic Student-t(3) (numpy generator, same shape and distribution as the GPU arm)",
        "config": dict(_config(args, thr, dens), density_note="density_a over the slab rows (row statistics are "
                       "exact per row); density_b from the slab's column statistics"),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cuda_library_loaded": "libxigemm_b200" in open("/proc/self/maps").read(),
    }
    print(json.dumps(line), flush=True)


def _config(args, thr, dens):
    c = {"workload": f"C3 xigemm M=N=K={args.m} Student-t(3) INT8 vector-wise AvgRule ~5% density"
                     if args.m == args.n == args.k == 8192 else
                     f"xigemm M={args.m} N={args.n} K={args.k} Student-t(3) INT8 vector-wise AvgRule",
         "m": args.m, "n": args.n, "k": args.k, "threshold_M": thr, "density_limit": 0.3,
         "scheme": "VectorWise", "policy": "AvgRule", "bits": 8, "rounding": "Nearest",
         "l2": "inputs (2 x 256 MiB) exceed the 126 MB L2; no flush needed"}
    if dens:
        c["density_a"], c["density_b"] = dens
    return c


def _roofline_block(m, n, k, rep, t, peaks, t_df, t_cp):
    """The bench's roofline object: whole call against SURVEY 8(d)'s summed
    2-term roofline (spec peaks; measured peaks beside), 3-term with the
    measured SIMT rate, and the dominant kernel's own algorithmic fraction."""
    rf = roofline(m, n, k, rep.nnz_a, rep.nnz_b, t)
    rm = roofline(m, n, k, rep.nnz_a, rep.nnz_b, t, peaks["int8_ops"], peaks["hbm_Bps"], peaks.get("idp4a_macs"))
    traffic = None
    try:  # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            tr = json.load(f)
        key = next(kk for kk in tr if kk.startswith("void k_gemm_i8_tc2<1, 4"))
        traffic = tr[key]
    except (OSError, KeyError, ValueError, StopIteration):
        pass
    # dominant kernel: the compensation launch (K4+K5).  Its algorithmic bytes:
    # A'q, RBq, RAq, B'q int8 in, D_F fp32 in, C fp32 out
    alg = 2 * (m * k + k * n) + 8 * m * n
    kern = {"name": "compensation launch (dr1 = A'q RBq, dr2 = RAq B'q, fused exact epilogue)",
            "ms": t_cp * 1e3, "algorithmic_bytes": alg,
            "algorithmic_GBps": alg / t_cp / 1e9, "frac_hbm": alg / t_cp / peaks["hbm_Bps"],
            "tensor_ops_issued": 4.0 * m * n * k, "tensor_tops": 4.0 * m * n * k / t_cp / 1e12,
            "frac_int8_peak": 4.0 * m * n * k / t_cp / peaks["int8_ops"],
            "d_f_gemm_ms": t_df * 1e3, "d_f_gemm_frac_int8_peak": 2.0 * m * n * k / t_df / peaks["int8_ops"]}
    if traffic:
        kern["dram_bytes"] = traffic.get("bytes_per_launch")
        kern["dram_over_algorithmic"] = traffic.get("bytes_per_launch", 0) / alg
        kern["traffic_source"] = traffic.get("source")
    return {
        "bound": "tensor+hbm",
        "model": "T_roof = 2MNK/P_i8 + B_alg/BW (SURVEY.md 8(d), summed); achieved = 2MNK/t, peak = 2MNK/T_roof, "
                 "frac = T_roof/t",
        "achieved": rf["achieved"], "peak": rf["peak"], "unit": "TFLOP/s", "frac": rf["frac"],
        "peak_source": "spec: P_i8 = 4.5e15 op/s, BW = 8.0e12 B/s",
        "t_roof_us": rf["t_roof_us"], "tensor_us": rf["tensor_us"], "hbm_us": rf["hbm_us"],
        "b_alg_bytes": rf["b_alg_bytes"],
        "measured_peaks": {"int8_tops": peaks["int8_ops"] / 1e12, "int8_source": peaks["int8_source"],
                           "hbm_GBps": peaks["hbm_Bps"] / 1e9, "hbm_source": peaks["hbm_source"],
                           "t_roof_us": rm["t_roof_us"], "peak": rm["peak"], "frac": rm["frac"]},
        "three_term": dict(rm.get("three_term", {}), p_simt_macs=peaks.get("idp4a_macs"),
                           p_imad_macs=peaks.get("imad_macs"),
                           note="adds (nnzA*N + nnzB*M) int8 MACs at the measured IDP4A rate; peaks measured"),
        "traffic": kern.get("dram_bytes"),
        "dominant_kernel": kern,
    }


def run_b200(args, world, rank, local):
    import numpy as np
    import torch
    import paper_2403_06924_b200 as xg

    torch.cuda.set_device(local)
    L = xg.lib()
    m, n, k = args.m, args.n, args.k
    a = xg.generate("student_t3", m, k, 1, 0.0, 1.0)
    b = xg.generate("student_t3", k, n, 2, 0.0, 1.0)
    scheme, policy = xg.QuantScheme.VectorWise, xg.ReductionPolicy.AvgRule
    thr = args.threshold
    if thr is None:
        thr = find_threshold(xg, a, b, scheme, policy)
    cfg = xg.XigemmConfig(threshold=thr, scheme=scheme, policy=policy)
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    rep = xg.xigemm(a, b, cfg=cfg, out=out)
    dens = (rep.density_a, rep.density_b)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        xg.xigemm(a, b, cfg=cfg, out=out)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    L.xg_launch_count(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gemm_ns = {"gemm_df": [], "gemm_comp": []}
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r = xg.xigemm(a, b, cfg=cfg, out=out)
            gemm_ns["gemm_df"].append(r.timings["gemm_df"])
            gemm_ns["gemm_comp"].append(r.timings["gemm_comp"])
        e1.record(stream)
        torch.cuda.synchronize()
    launches = int(L.xg_launch_count(1))
    ms = e0.elapsed_time(e1) / args.steps
    barrier()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ops = 2.0 * m * n * k
    value = ops * world / (ms * 1e-3) / 1e12

    # ---- e2e through the host-buffer C-ABI call (pinned host buffers) ----
    e2e_val = e2e_pageable = None
    if not args.no_e2e:
        ah = torch.empty((m, k), dtype=torch.float32, pin_memory=True)
        bh = torch.empty((k, n), dtype=torch.float32, pin_memory=True)
        oh = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
        ah.copy_(a)
        bh.copy_(b)
        an, bn, on = ah.numpy(), bh.numpy(), oh.numpy()
        for _ in range(2):
            xg.xigemm_host(an, bn, cfg=cfg, out=on)
        e2e_steps = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            xg.xigemm_host(an, bn, cfg=cfg, out=on)
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([e2e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e_val = ops * world / e2e_s / 1e12
        # host path result equals the device path result
        assert np.array_equal(on.view(np.uint32), out.cpu().numpy().view(np.uint32))
        # the same call on pageable buffers (plain numpy, like the C++ drop-in's
        # std::vector memory): xg_xigemm_host stages them through pinned slots
        ap, bp, op = an.copy(), bn.copy(), np.empty_like(on)
        del ah, bh, oh
        xg.xigemm_host(ap, bp, cfg=cfg, out=op)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            xg.xigemm_host(ap, bp, cfg=cfg, out=op)
        pg_s = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([pg_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pg_s = float(t.item())
        e2e_pageable = ops * world / pg_s / 1e12
        assert np.array_equal(op.view(np.uint32), out.cpu().numpy().view(np.uint32))
        del ap, bp, op

    if rank != 0:
        return
    # ---- CPU baseline (1 core, background thread: the reference releases the GIL) ----
    cpu_thread, cpu_res = None, {}
    if not args.no_cpu_baseline:
        jobs = []
        for nm, sz, kind_, lo, hi, target in (("C1", 1024, "uniform", -1.0, 1.0, 0.05),
                                              ("C2", 4096, "normal", 0.0, 1.0, 0.05)):
            if nm == "C2" and args.cpu_quick:
                continue
            x = xg.generate(kind_, sz, sz, 1, lo, hi)
            y = xg.generate(kind_, sz, sz, 2, lo, hi)
            th = find_threshold(xg, x, y, scheme, policy, target)
            g = xg.xigemm(x, y, cfg=xg.XigemmConfig(threshold=th, scheme=scheme, policy=policy))
            jobs.append(dict(name=nm, a=x.cpu().numpy(), b=y.cpu().numpy(), thr=th, scheme=1, policy=0,
                             gpu_out=g.result.cpu().numpy(), mode="full", reps=3 if nm == "C1" else 1,
                             gpu_density=(g.density_a, g.density_b)))
        jobs.append(dict(name="C3", a=a[:2048].cpu().numpy(), b=b.cpu().numpy(), thr=thr, scheme=1, policy=0,
                         mode="fit"))

        def cpu_work():
            try:
                cpu_res.update(cpu_baseline_run(jobs))
            except Exception as ex:  # noqa: BLE001
                cpu_res["error"] = str(ex)[:300]

        cpu_thread = threading.Thread(target=cpu_work, daemon=True)
        cpu_thread.start()

    peaks = measure_peaks(L)
    t_df = float(np.mean(gemm_ns["gemm_df"])) * 1e-9
    t_cp = float(np.mean(gemm_ns["gemm_comp"])) * 1e-9
    roof = _roofline_block(m, n, k, rep, ms * 1e-3, peaks, t_df, t_cp)
    # live reference point: cuBLASLt int8 GEMM (torch._int_mm, s32 out, no epilogue) at the
    # same shape - a library call for context, never on the product path
    try:
        ia = torch.randint(-127, 128, (m, k), dtype=torch.int8, device="cuda")
        ib = torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(ia, ib)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(10):
            torch._int_mm(ia, ib)
        c1.record()
        torch.cuda.synchronize()
        roof["dominant_kernel"]["cublaslt_int8_tops_same_shape"] = ops / (c0.elapsed_time(c1) / 10 * 1e-3) / 1e12
        del ia, ib
    except Exception:  # noqa: BLE001
        pass
    # accuracy (BASELINE.json metric, second half): e_delta = ||C64 - C||_F / ||C64||_F
    # against an FP64 GEMM of the same inputs (metrics.cpp:7-33), for xigemm and the
    # paper's two baselines
    accuracy = None
    if not args.no_accuracy:
        try:
            c64 = a.double() @ b.double()
            nref = torch.linalg.norm(c64)

            def e_delta(x):
                return float(torch.linalg.norm(c64 - x.double()) / nref)

            accuracy = {"reference": "FP64 GEMM of the same fp32 inputs (torch float64 matmul on the GPU)",
                        "e_delta_xigemm": e_delta(out),
                        "e_delta_origin": e_delta(xg.quantized_gemm_direct(a, b, cfg)),
                        "e_delta_full_residual": e_delta(xg.quantized_gemm_full_residual(a, b, cfg)),
                        "e_delta_fp32_gemm": e_delta(a @ b)}
            del c64
        except Exception as ex:  # noqa: BLE001
            accuracy = {"error": str(ex)[:200]}
    del a, b
    torch.cuda.empty_cache()
    configs = None if args.no_configs else run_configs(xg, torch, peaks, args.steps)
    cpu = None
    if cpu_thread is not None:
        cpu_thread.join()
        c3 = cpu_res.get("C3", {})
        if "seconds" in c3:
            cpu = {"value": 2.0 * m * n * k / c3["seconds"] / 1e12, "unit": "TFLOP/s", "cores": 1,
                   "kind": cpu_res.get("kind"),
                   "sample": "C3: the reference's xigemm (oracle/_ref) on 16- and 48-row slabs of the same A "
                             "against the full B, one core; t = t_B + M*t_row (estimate). C1 and C2: full "
                             "problems on the GPU arm's inputs (outputs compared bit for bit)",
                   "configs": cpu_res}
        else:
            cpu = {"value": None, "unit": "TFLOP/s", "cores": 1, "kind": cpu_res.get("kind"), "configs": cpu_res}
    line = {
        "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8 (fp64/fp32 exact epilogues)",
        "data": "synthetic Student-t(3) (device SplitMix64 generator), seeds A=1 B=2",
        "config": _config(args, thr, dens),
        "e2e": {"value": e2e_val, "unit": "TFLOP/s",
                "h2d_bytes_per_step": 4 * (m * k + k * n), "d2h_bytes_per_step": 4 * m * n,
                "buffers": "pinned host memory (torch pin_memory), xg_xigemm_host",
                "pageable": {"value": e2e_pageable, "unit": "TFLOP/s",
                             "buffers": "pageable numpy arrays - the C++ drop-in's std::vector memory - staged "
                                        "through pinned slots inside xg_xigemm_host"}} if e2e_val else None,
        "roofline": roof,
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "accuracy": accuracy,
        "stage_ns": {kk: int(vv) for kk, vv in r.timings.items()},  # last timed call
        "configs": configs,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def run_b200_sharded(args, world, rank, local):
    """--gpus N > 1: the row-sharded pipeline.  Weak
    scaling: every rank owns an M-row block of a tall A (M*N_gpus x K) and of C;
    B (K x N) lives on rank 0 and is replicated by one NCCL broadcast inside
    every timed step; the exact couplings (max|A|, max|RA|, column statistics,
    nnz(A')) are NCCL all-reduces between the pipeline stages."""
    import torch
    import torch.distributed as dist
    import paper_2403_06924_b200 as xg
    from paper_2403_06924_b200 import sharded

    # local % device count: the one-box check of this path runs both ranks on one
    # GPU over gloo (XG_BENCH_BACKEND=gloo); one process per GPU otherwise
    torch.cuda.set_device(local % torch.cuda.device_count())
    m, n, k = args.m, args.n, args.k
    a = xg.generate("student_t3", m, k, 1 + 7919 * rank, 0.0, 1.0)
    b = xg.generate("student_t3", k, n, 2, 0.0, 1.0) if rank == 0 else \
        torch.empty((k, n), dtype=torch.float32, device="cuda")
    sharded.broadcast_b(b)
    scheme, policy = xg.QuantScheme.VectorWise, xg.ReductionPolicy.AvgRule
    t = torch.tensor([args.threshold or 0.0], dtype=torch.float64, device="cuda")
    if args.threshold is None and rank == 0:
        t[0] = find_threshold(xg, a, b, scheme, policy)
    dist.broadcast(t, src=0)
    thr = float(t.item())
    cfg = xg.XigemmConfig(threshold=thr, scheme=scheme, policy=policy)
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")

    def step():
        sharded.broadcast_b(b)
        # graph capture needs NCCL collectives (the gloo check runs eagerly)
        return sharded.xigemm_sharded(a, b, cfg=cfg, out=out, rank_rows=[m] * world,
                                      graph=dist.get_backend() == "nccl")

    rep = step()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    sharded.launch_count(reset=True)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            rep = step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = sharded.launch_count(reset=True)  # includes the kernels replayed in the shard's graph
    tt = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    ops = 2.0 * m * world * n * k
    value = ops / (ms * 1e-3) / 1e12
    # SURVEY 8(e)'s resident-B design beside it: B already on every rank (weights
    # style), the same step without the broadcast
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        sharded.xigemm_sharded(a, b, cfg=cfg, out=out, rank_rows=[m] * world, graph=dist.get_backend() == "nccl")
    e1.record(stream)
    torch.cuda.synchronize()
    tr = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(tr, op=dist.ReduceOp.MAX)
    ms_res = float(tr.item())
    sharded.launch_count(reset=True)

    # e2e: host A rows on every rank, host B on rank 0, C rows back to the host
    ah = torch.empty((m, k), dtype=torch.float32, pin_memory=True)
    ah.copy_(a)
    bh = torch.empty((k, n), dtype=torch.float32, pin_memory=True)
    if rank == 0:
        bh.copy_(b)
    oh = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
    ad = torch.empty_like(a)
    bd = torch.empty_like(b)

    def e2e_step():
        ad.copy_(ah, non_blocking=True)
        if rank == 0:
            bd.copy_(bh, non_blocking=True)
        sharded.broadcast_b(bd)
        sharded.xigemm_sharded(ad, bd, cfg=cfg, out=out, rank_rows=[m] * world, graph=dist.get_backend() == "nccl")
        oh.copy_(out, non_blocking=True)
        torch.cuda.synchronize()

    e2e_step()
    dist.barrier()
    n_e2e = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        e2e_step()
    te = torch.tensor([(time.perf_counter() - t0) / n_e2e], device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = ops / float(te.item()) / 1e12
    if rank != 0:
        return
    # roofline of one rank's share: its M rows against the replicated B (the
    # B-side stages run on every rank: B_alg counts them once per rank)
    rf = roofline(m, n, k, rep.nnz_a // world, rep.nnz_b, ms * 1e-3)
    peaks = measure_peaks(xg.lib())
    rm = roofline(m, n, k, rep.nnz_a // world, rep.nnz_b, ms * 1e-3, peaks["int8_ops"], peaks["hbm_Bps"],
                  peaks.get("idp4a_macs"))
    cpu = None
    if not args.no_cpu_baseline:
        c3 = cpu_baseline_run([dict(name="C3", a=a[:2048].cpu().numpy(), b=b.cpu().numpy(), thr=thr, scheme=1,
                                    policy=0, mode="fit")]).get("C3", {})
        if "seconds" in c3:
            cpu = {"value": 2.0 * m * n * k / c3["seconds"] / 1e12, "unit": "TFLOP/s", "cores": 1,
                   "kind": "reference", "sample": "one rank's C3 rows: two-slab fit of xigemm_ref (16/48 rows), "
                                                  "t = t_B + M*t_row (estimate)", "fit": c3}
    line = {
        "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8 (fp64/fp32 exact epilogues)",
        "data": "synthetic Student-t(3) (device SplitMix64 generator), A rows seeded per rank, B seed 2",
        "config": dict(_config(args, thr, (rep.density_a, rep.density_b)),
                       workload=f"row-sharded xigemm: A {m * world}x{k} ({m} rows per GPU), B {k}x{n} "
                                f"broadcast from rank 0 every step, Student-t(3), INT8 vector-wise AvgRule",
                       parallelism=f"rows{world} (B replicated by NCCL broadcast; exact all-reduce couplings)"),
        "variants": {
            "resident_b": {"value": ops / (ms_res * 1e-3) / 1e12, "ms_per_step": ms_res,
                           "note": "B resident on every rank (SURVEY 8(e) resident-B design): the step without "
                                   "the broadcast"},
            "column_sliced_b": "not built: SURVEY 8(e)'s scalable design (1/g column slice of the B side per "
                               "rank, all-gather of Bq / RBq / B'q) - the broadcast design is the north star's"},
        "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": 4 * (m * k * world + k * n),
                "d2h_bytes_per_step": 4 * m * n * world},
        "roofline": {"bound": "tensor+hbm", "model": "per rank: T_roof = 2MNK/P_i8 + B_alg/BW of its rows "
                     "(B-side stages counted on every rank); frac = T_roof / t", "achieved": rf["achieved"],
                     "peak": rf["peak"], "unit": "TFLOP/s per GPU", "frac": rf["frac"],
                     "peak_source": "spec: P_i8 = 4.5e15 op/s, BW = 8.0e12 B/s", "t_roof_us": rf["t_roof_us"],
                     "measured_peaks": {"frac": rm["frac"], "t_roof_us": rm["t_roof_us"]},
                     "three_term": rm.get("three_term"), "traffic": None},
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--m", type=int, default=M_DEFAULT)
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--k", type=int, default=K_DEFAULT)
    ap.add_argument("--threshold", type=float, default=None)
    ap.add_argument("--ref-rows", type=int, default=None, help="--impl reference: tiny slabs (<= 4: 2/6 rows)")
    ap.add_argument("--ref-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-quick", action="store_true", help="cpu_baseline without the full C2 problem (~60 s)")
    ap.add_argument("--no-configs", action="store_true", help="only the headline configuration")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    ap.add_argument("--no-accuracy", action="store_true", help="skip the FP64-GEMM error report")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent full problems per GPU instead of the row-sharded pipeline")
    ap.add_argument("--sharded", action="store_true",
                    help="use the row-sharded pipeline even at N=1 (needs torchrun / a process group)")
    args = ap.parse_args()
    args.ref_rows_set = args.ref_rows is not None
    if args.impl == "reference":  # CPU only: rank 0 runs it, the other ranks exit 0; no process group
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = _dist_init()
    if (world > 1 and not args.replicas) or args.sharded:
        run_b200_sharded(args, world, rank, local)
    else:
        run_b200(args, world, rank, local)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
