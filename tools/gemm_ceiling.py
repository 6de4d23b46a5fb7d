"""MMA-pipeline ceiling probe: DF GEMM 8192^3 with TMA loads and/or epilogue disabled."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06924_b200 as xg
L = xg.lib()
L.xg_debug_gemm_df.restype = ctypes.c_double
L.xg_debug_gemm_df.argtypes = [ctypes.c_int] * 5
n = 8192
for flags, name in [(16, "zeros full"), (18, "zeros no-epi"), (0, "random full"), (2, "random no-epi"), (1, "random no-TMA"), (3, "random MMA only")]:
    ms = L.xg_debug_gemm_df(n, n, n, flags, 10)
    print(f"{name:14s} {ms:.3f} ms  {2 * n**3 / ms / 1e9:.0f} TOPS", flush=True)
