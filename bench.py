"""Benchmark of the compensated INT8 GEMM (arXiv 2403.06924 "xigemm") on B200.

One step = one full xigemm() over one synthetic batch: quantize A and B,
tcgen05 INT8 GEMM, |D_F| statistics, residual quantisation + threshold
selection, compensation GEMM with the fused epilogue.  Metric (BASELINE.json):
effective TFLOP/s = 2MNK / t.

Workload (default): C3 of BASELINE.json — M=N=K=8192, Student-t(3) FP32 inputs,
INT8 vector-wise quantisation, AvgRule, threshold M bisected for ~5% residual
density (s = 0.3 so the sparse path is taken).  Inputs (256 MiB each) exceed the
126 MB L2, so no explicit flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU (torchrun, --gpus N > 1): the row-sharded pipeline (weak scaling:
M rows of A and C per GPU, B broadcast from rank 0 by NCCL every step, exact
all-reduce couplings between the stages; paper_2403_06924_b200/sharded.py).
--replicas runs N independent full problems instead.
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


def _dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or "MASTER_ADDR" in os.environ:
        import torch
        import torch.distributed as dist
        backend = "nccl" if os.environ.get("XG_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
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


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    except OSError:
        return 6650.0, 1590.0, "fallback"


def find_threshold(xg, a, b, scheme, policy, target=TARGET_DENSITY):
    """Bisects M (log scale) so max(density_a, density_b) is within 10% of target."""
    lo, hi = 1e-4, 10.0
    best = None
    for _ in range(30):
        mid = (lo * hi) ** 0.5
        cfg = xg.XigemmConfig(threshold=mid, scheme=scheme, policy=policy)
        rep = xg.xigemm(a, b, cfg=cfg)
        d = max(rep.density_a, rep.density_b)
        best = (mid, rep.density_a, rep.density_b)
        if abs(d - target) <= 0.1 * target:
            break
        if d > target:
            lo = mid
        else:
            hi = mid
    return best


def cpu_baseline_sample(a_host, b_host, thr, rows, threads=1, reps=1):
    """The reference's xigemm (oracle/_ref, else the C restatement) on a row slab
    of the same A against the full B, on host cores.  Returns (ops/s, seconds, kind)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracle_lib as ol
    r = ol.reference()
    kind = "reference"
    if r is None:
        r, kind = ol.oracle(), "port"
    cfg = ol.cfg(threshold=thr, density_limit=0.3, scheme=1, policy=0, rounding=1)
    k, n = b_host.shape
    slabs = [np.ascontiguousarray(a_host[(t * rows) % a_host.shape[0]:][:rows]) for t in range(threads)]
    outs = [None] * threads

    def work(t):
        outs[t] = r.xigemm(slabs[t], b_host, config=cfg)

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
    ops = 2.0 * rows * n * k * threads
    return ops / best, best, kind


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU implementation on this box's host
    cores (all of them), on the same metric/config; bounded row-slab samples."""
    import numpy as np
    if world > 1 and rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol
    m, n, k = args.m, args.n, args.k
    threads = min(os.cpu_count() or 1, 32)
    try:
        import psutil
        threads = max(1, min(threads, int(psutil.virtual_memory().available / 2.0e9)))
    except Exception:  # noqa: BLE001
        pass
    # inputs: same generator stream as the GPU arm (device generator), host copy
    import torch
    import paper_2403_06924_b200 as xg
    if torch.cuda.is_available():
        a = xg.generate("student_t3", m, k, 1, 0.0, 1.0).cpu().numpy()
        b = xg.generate("student_t3", k, n, 2, 0.0, 1.0).cpu().numpy()
        thr = args.threshold or find_threshold(xg, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                                               xg.QuantScheme.VectorWise, xg.ReductionPolicy.AvgRule)[0]
    else:  # no GPU on this host: same distribution from numpy
        rng = np.random.default_rng(1)
        z = rng.standard_normal((m, k), dtype=np.float32)
        a = (z / np.sqrt((rng.standard_normal((m, k), dtype=np.float32) ** 2 * 3) / 3)).astype(np.float32)
        b = a.T.copy()
        thr = args.threshold or 0.01
    # larger slabs than the single-core baseline: the reference redoes all of
    # B's quantisation per call, which a 16-row slab would over-weight
    # exactly --steps K steps (or --ref-steps); each a bounded sample: 64-row
    # slabs (~4-5 s per step on the GPU box's cores), smaller beyond 30 steps so
    # the whole run stays within a few minutes
    nsteps = max(1, args.steps if args.ref_steps is None else args.ref_steps)
    rows = args.ref_rows if args.ref_rows_set else (64 if nsteps <= 30 else max(8, 64 * 30 // nsteps))
    vals = []
    for _ in range(args.warmup):
        pass  # CPU: no warm-up effect worth paying minutes for
    for _ in range(nsteps):
        v, dt, kind = cpu_baseline_sample(a, b, thr, rows, threads=threads)
        vals.append((v, dt))
    value = sorted(v for v, _ in vals)[len(vals) // 2] / 1e12
    step_s = sorted(dt for _, dt in vals)[len(vals) // 2]
    line = {
        "impl": "reference", "metric": "effective TFLOP/s (2MNK/t) of compensated GEMM",
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": len(vals),
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8/fp64 (reference CPU)",
        "data": "synthetic Student-t(3)",
        "config": _config(args, thr, None),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": kind,
                         "sample": f"{threads} threads x xigemm_ref on a {rows}-row slab of A "
                                   f"against the full {k}x{n} B per step"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
        thr = find_threshold(xg, a, b, scheme, policy)[0]
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
    e2e_val = None
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

    if rank != 0:
        return
    hbm, bf16, src = _peaks()
    int8_peak = 2.0 * bf16  # dense INT8 = 2x dense bf16 on B200 (proxy for the missing INT8 figure)
    t_df = float(np.mean(gemm_ns["gemm_df"])) * 1e-9
    t_cp = float(np.mean(gemm_ns["gemm_comp"])) * 1e-9
    # dominant kernel: the larger of the two tensor-core launches
    if t_cp >= t_df:
        name, kops, tk = ("compensation GEMM (one launch, masked-dense dr1 and dr2 per tile: 4MNK tensor ops)",
                          4.0 * m * n * k, t_cp)
    else:
        name, kops, tk = "D_F GEMM (2MNK tensor ops)", 2.0 * m * n * k, t_df
    achieved = kops / tk / 1e12
    traffic = None
    try:  # DRAM bytes per launch of that kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "r1k_gemm_traffic.json")) as f:
            tr = json.load(f)
        pre = "void k_gemm_i8_tc2<1, 4, 1" if t_cp >= t_df else "void k_gemm_i8_tc2<1, 1, 1"
        key = next(kk for kk in tr if kk.startswith(pre))
        traffic = {"dram_bytes_per_launch": tr[key]["bytes_per_launch"],
                   # int8 operands in (A'q, RBq, RAq, B'q | Aq, Bq), fp32 D_F in (compensation), fp32 out
                   "algorithmic_bytes_per_launch": (2 * (m * k + k * n) + 8 * m * n) if t_cp >= t_df
                   else (m * k + k * n + 4 * m * n),
                   "source": "profiles/r1k_gemm_traffic.json (ncu --set full, this kernel, C3)"}
    except (OSError, KeyError, ValueError, StopIteration):
        pass
    # live reference point for the INT8 denominator (MEASURED_PEAKS.json has
    # bf16 only): cuBLASLt int8 GEMM (torch._int_mm, s32 out, no epilogue) at
    # the same shape; library call for context, never on the product path
    cublaslt = None
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
        cublaslt = 2.0 * m * n * k / (c0.elapsed_time(c1) / 10 * 1e-3) / 1e12
        del ia, ib
    except Exception:  # noqa: BLE001
        pass
    # accuracy (BASELINE.json metric, second half): relative Frobenius error
    # e_delta = ||C64 - C||_F / ||C64||_F against an FP64 GEMM of the same
    # inputs (metrics.cpp:7-33), for xigemm and the paper's two baselines
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
    cpu = None
    if not args.no_cpu_baseline:
        v, dt, kind = cpu_baseline_sample(a.cpu().numpy(), b.cpu().numpy(), thr, args.ref_rows, 1)
        cpu = {"value": v / 1e12, "unit": "TFLOP/s", "cores": 1, "kind": kind,
               "sample": f"xigemm_ref on a {args.ref_rows}-row slab of A against the full "
                         f"{k}x{n} B ({dt:.1f} s); 2*rows*N*K/t"}
    line = {
        "metric": "effective TFLOP/s (2MNK/t) of compensated GEMM",
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8 (fp64/fp32 exact epilogues)",
        "data": "synthetic Student-t(3) (device SplitMix64 generator), seeds A=1 B=2",
        "config": _config(args, thr, dens),
        "e2e": {"value": e2e_val, "unit": "TFLOP/s",
                "h2d_bytes_per_step": 4 * (m * k + k * n), "d2h_bytes_per_step": 4 * m * n} if e2e_val else None,
        "roofline": {"bound": "tensor", "kernel": name, "achieved": achieved,
                     "peak": int8_peak, "unit": "TFLOP/s", "frac": achieved / int8_peak,
                     # dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full)
                     "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                     "traffic_detail": traffic,
                     "peak_source": f"2 x bf16_tflops ({bf16}) of MEASURED_PEAKS.json ({src}); INT8 dense = 2x bf16 on B200",
                     "gemm_df_ms": t_df * 1e3, "gemm_comp_ms": t_cp * 1e3,
                     "cublaslt_int8_tflops": cublaslt,
                     "frac_of_cublaslt_int8": (achieved / cublaslt) if cublaslt else None},
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "accuracy": accuracy,
        "stage_ns": {kk: int(vv) for kk, vv in r.timings.items()},  # last timed call
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
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2403_06924_b200 as xg
    from paper_2403_06924_b200 import sharded

    torch.cuda.set_device(local)
    m, n, k = args.m, args.n, args.k
    a = xg.generate("student_t3", m, k, 1 + 7919 * rank, 0.0, 1.0)
    b = xg.generate("student_t3", k, n, 2, 0.0, 1.0) if rank == 0 else \
        torch.empty((k, n), dtype=torch.float32, device="cuda")
    sharded.broadcast_b(b)
    scheme, policy = xg.QuantScheme.VectorWise, xg.ReductionPolicy.AvgRule
    t = torch.tensor([args.threshold or 0.0], dtype=torch.float64, device="cuda")
    if args.threshold is None and rank == 0:
        t[0] = find_threshold(xg, a, b, scheme, policy)[0]
    dist.broadcast(t, src=0)
    thr = float(t.item())
    cfg = xg.XigemmConfig(threshold=thr, scheme=scheme, policy=policy)
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")

    def step():
        sharded.broadcast_b(b)
        return sharded.xigemm_sharded(a, b, cfg=cfg, out=out, rank_rows=[m] * world)

    rep = step()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    L = xg.lib()
    L.xg_launch_count(1)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = int(L.xg_launch_count(1))
    tt = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    ops = 2.0 * m * world * n * k
    value = ops / (ms * 1e-3) / 1e12

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
        sharded.xigemm_sharded(ad, bd, cfg=cfg, out=out, rank_rows=[m] * world)
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
    line = {
        "metric": "effective TFLOP/s (2MNK/t) of compensated GEMM",
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int8 (fp64/fp32 exact epilogues)",
        "data": "synthetic Student-t(3) (device SplitMix64 generator), A rows seeded per rank, B seed 2",
        "config": dict(_config(args, thr, (rep.density_a, rep.density_b)),
                       workload=f"row-sharded xigemm: A {m * world}x{k} ({m} rows per GPU), B {k}x{n} "
                                f"broadcast from rank 0 every step, Student-t(3), INT8 vector-wise AvgRule",
                       parallelism=f"rows{world} (B replicated by NCCL broadcast; exact all-reduce couplings)"),
        "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": 4 * (m * k * world + k * n),
                "d2h_bytes_per_step": 4 * m * n * world},
        "roofline": None,
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
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
    ap.add_argument("--ref-rows", type=int, default=None,
                    help="row slab of the CPU samples (default 16 for cpu_baseline, 64 for --impl reference)")
    ap.add_argument("--ref-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    ap.add_argument("--no-accuracy", action="store_true", help="skip the FP64-GEMM error report")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent full problems per GPU instead of the row-sharded pipeline")
    ap.add_argument("--sharded", action="store_true",
                    help="use the row-sharded pipeline even at N=1 (needs torchrun / a process group)")
    args = ap.parse_args()
    args.ref_rows_set = args.ref_rows is not None
    if args.ref_rows is None:
        args.ref_rows = 16
    world, rank, local = _dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif (world > 1 and not args.replicas) or args.sharded:
        run_b200_sharded(args, world, rank, local)
    else:
        run_b200(args, world, rank, local)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
