"""Print the mismatches of the epilogue dequantisation (xg_debug_dq_ff) against
float(p / (la*lb)) for the extreme-scale case of tests/test_gpu_parity.py."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_parity as t
rng = np.random.default_rng(99)
n = 1 << 20
p = np.concatenate([rng.integers(-300, 300, n // 2, dtype=np.int64),
                    rng.integers(-2**31, 2**31, n // 4, dtype=np.int64),
                    np.left_shift(1, rng.integers(0, 31, n // 4)) * rng.choice([-1, 1], n // 4)])
p = np.clip(p, -2**31, 2**31 - 1).astype(np.int32)
ea = rng.uniform(-53, 53, n)
eb = rng.uniform(-53, 53, n)
la = np.exp2(ea)
lb = np.exp2(eb)
la[: n // 8] = np.exp2(np.round(ea[: n // 8]))
lb[n // 8: n // 4] = np.exp2(np.round(eb[n // 8: n // 4]))
got, flags = t._dq_ff(p, la, lb)
ref = t._dq_ref(p, la, lb)
bad = np.nonzero(got.view(np.uint32) != ref.view(np.uint32))[0]
print("mismatches", len(bad), "of", n)
for i in bad[:30]:
    print(i, p[i], repr(la[i]), repr(lb[i]), "1/la", 1 / la[i], "1/lb", 1 / lb[i], "got", got[i], "ref", ref[i], "flag", flags[i])
