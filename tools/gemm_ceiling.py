"""MMA-pipeline ceiling probe: DF GEMM 8192^3 with TMA loads and/or epilogue
disabled (debug flags of k_gemm_i8_tc2), with SM clock / power sampled by NVML
during each configuration."""
import ctypes, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06924_b200 as xg
import pynvml
L = xg.lib()
L.xg_debug_gemm_df.restype = ctypes.c_double
L.xg_debug_gemm_df.argtypes = [ctypes.c_int] * 5
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))))
        time.sleep(0.002)


n = int(os.environ.get("N", "8192"))
shape = tuple(int(v) for v in os.environ.get("SHAPE", f"{n},{n},{n}").split(","))  # M,N,K
iters = int(os.environ.get("ITERS", "200"))
cfgs = [(16, "zeros full"), (18, "zeros no-epi"), (0, "random full"), (2, "random no-epi"),
        (1, "random no-TMA"), (3, "random MMA only"), (4, "random ld-only epi"), (8, "random no-store"),
        (32, "random no-MMA"), (34, "TMA only"), (64, "no-math"), (72, "no-math no-store"),
        (128, "fp32 math"), (33, "epilogue only"), (41, "epi only no-store"), (97, "epi only no-math"),
        (37, "epi only TMEM drain")]
sel = os.environ.get("CFGS")
if sel:
    cfgs = [c for c in cfgs if str(c[0]) in sel.split(",")]
for flags, name in cfgs:
    time.sleep(float(os.environ.get("GAP", "0")))
    stop, smp = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, smp))
    th.start()
    ms = L.xg_debug_gemm_df(*shape, flags, iters)
    stop.set()
    th.join()
    mid = smp[len(smp) // 4: 3 * len(smp) // 4] or smp
    clk = sorted(s[0] for s in mid)[len(mid) // 2] if mid else 0
    pw = sorted(s[1] for s in mid)[len(mid) // 2] if mid else 0
    rs = 0
    for s in mid:
        rs |= s[2]
    print(f"{name:18s} {ms:.3f} ms  {2 * shape[0] * shape[1] * shape[2] / ms / 1e9:5.0f} TOPS  sm {clk} MHz  {pw:.0f} W  reasons 0x{rs:x}",
          flush=True)
