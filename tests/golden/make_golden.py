"""Regenerates tests/golden/*.npz from the REFERENCE itself.

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py
Every expected value stored here comes out of oracle/_ref/libxigemm_ref.so,
i.e. the unmodified reference sources compiled by oracle/Makefile.  Inputs are
SplitMix64 streams (test_support.hpp:16-24) so they are regenerable too, but
they are stored alongside for clarity.  tests/test_oracle.py pins the C
restatement to these files; tests/test_gpu_parity.py pins the CUDA path.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as ol  # noqa: E402

# (m, k, n, seed_a, seed_b, lo, hi)
SHAPES = [(1, 1, 1, 3, 4, -1.0, 1.0), (3, 3, 3, 5, 6, -2.0, 2.0), (24, 20, 28, 1, 2, -3.0, 3.0),
          (33, 17, 29, 7, 8, -10.0, 10.0), (5, 130, 7, 9, 10, -1.0, 1.0),
          (64, 64, 64, 11, 12, -1.0, 1.0), (129, 96, 200, 13, 14, -4.0, 4.0)]
# (threshold, density_limit, scheme, policy, rounding, bits)
CONFIGS = [(0.5, 0.3, 0, 1, 1, 8), (0.05, 0.3, 1, 0, 1, 8), (0.3, 0.5, 1, 1, 0, 8),
           (1e-30, 0.5, 0, 0, 1, 8), (1e9, 0.5, 1, 0, 1, 8), (0.2, 1.0, 0, 0, 0, 4),
           (0.08, 0.2, 1, 0, 1, 4)]


def main():
    ref = ol.reference()
    assert ref is not None, "build oracle/_ref first (make -C oracle ref)"
    cases = {}
    idx = 0
    for (m, k, n, sa, sb, lo, hi) in SHAPES:
        a = ol.random_dense(m, k, sa, lo, hi)
        b = ol.random_dense(k, n, sb, lo, hi)
        for (thr, s, scheme, pol, rnd, bits) in CONFIGS:
            c = ol.cfg(bits=bits, threshold=thr, density_limit=s, scheme=scheme, policy=pol,
                       rounding=rnd)
            rc, out, rep = ref.xigemm(a, b, config=c)
            assert rc == 0
            rc2, full, _ = ref.xigemm(a, b, config=c, reduce=False)
            rc3, direct = ref.gemm_direct(a, b, config=c)
            assert rc2 == 0 and rc3 == 0
            key = f"case{idx:03d}"
            cases[key + "_meta"] = np.array([m, k, n, sa, sb, scheme, pol, rnd, bits, rep.path,
                                             SHAPES.index((m, k, n, sa, sb, lo, hi))], np.int64)
            cases[key + "_fmeta"] = np.array([lo, hi, thr, s, rep.density_a, rep.density_b])
            cases[f"shape{SHAPES.index((m, k, n, sa, sb, lo, hi))}_a"] = a
            cases[f"shape{SHAPES.index((m, k, n, sa, sb, lo, hi))}_b"] = b
            cases[key + "_xigemm"] = out
            cases[key + "_full"] = full
            cases[key + "_direct"] = direct
            idx += 1
    np.savez_compressed(os.path.join(HERE, "pipeline_golden.npz"), **cases)

    # Stage intermediates (pipeline.cpp:44-149 replayed through the reference's
    # own stage functions) for a few cases.
    stages = {}
    for j, (m, k, n, sa, sb, lo, hi) in enumerate(SHAPES[2:6]):
        a = ol.random_dense(m, k, sa, lo, hi)
        b = ol.random_dense(k, n, sb, lo, hi)
        for ci, (thr, s, scheme, pol, rnd, bits) in enumerate(CONFIGS[:3]):
            c = ol.cfg(bits=bits, threshold=thr, density_limit=s, scheme=scheme, policy=pol,
                       rounding=rnd)
            rc, d = ref.dump(a, b, c)
            assert rc == 0
            pre = f"s{j}_{ci}_"
            stages[pre + "cfg"] = np.array([thr, s, scheme, pol, rnd, bits], np.float64)
            stages[pre + "a"] = a
            stages[pre + "b"] = b
            for name, arr in d.items():
                stages[pre + name] = arr
    np.savez_compressed(os.path.join(HERE, "stages_golden.npz"), **stages)

    # Scalar / small known answers straight from the reference API.
    ka = {}
    for bits in (4, 8):
        for rnd in (0, 1):
            for scheme in (0, 1, 2):
                x = ol.random_dense(9, 7, 100 + bits + rnd + scheme, -5, 5)
                rc, q, sc = ref.quantize(x, bits, scheme, rnd)
                ka[f"q_{bits}_{rnd}_{scheme}_in"] = x
                ka[f"q_{bits}_{rnd}_{scheme}_q"] = q
                ka[f"q_{bits}_{rnd}_{scheme}_s"] = sc
    # quantize_with_scales with a huge scale: the reference's out-of-range llround
    x = np.array([[1.0, -2.0, 3.0e-3, 0.0]], np.float32)
    for rnd in (0, 1):
        rc, q = ref.quantize_with_scales(x, np.array([1e300]), 8, 0, rnd)
        ka[f"huge_{rnd}"] = q
    np.savez_compressed(os.path.join(HERE, "known_answers.npz"), **ka)
    print("wrote", idx, "pipeline cases")


if __name__ == "__main__":
    main()
