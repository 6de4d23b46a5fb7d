"""Pins the C restatement (oracle/xigemm_oracle.c) before it is trusted as the
parity oracle: (1) known answers from the reference's own suites, (2) the
golden vectors generated from the reference itself (tests/golden/), (3) live
bit-for-bit comparison against oracle/_ref when that build exists."""
import numpy as np
import pytest

import oracle_lib as ol

GOLD = ol.os.path.join(ol.ROOT, "tests", "golden")


def bits_eq(x, y):
    x = np.asarray(x)
    y = np.asarray(y)
    if x.dtype.kind == "f":
        return x.shape == y.shape and np.array_equal(x.view(np.uint32 if x.dtype == np.float32 else np.uint64),
                                                     y.view(np.uint32 if y.dtype == np.float32 else np.uint64))
    return np.array_equal(x, y)


# ---- known answers (reference test suites) --------------------------------
def test_compute_scale_known(oracle):
    import ctypes as C
    out = C.c_double(0)
    oracle.lib.xo_compute_scale.argtypes = [C.c_double, C.c_int, C.POINTER(C.c_double)]
    assert oracle.lib.xo_compute_scale(4.0, 8, C.byref(out)) == 0 and abs(out.value - 31.75) < 1e-12  # test_quant.cpp:19-25
    assert oracle.lib.xo_compute_scale(0.0, 8, C.byref(out)) == 0 and out.value == 1.0
    assert oracle.lib.xo_compute_scale(4.0, 4, C.byref(out)) == 0 and abs(out.value - 1.75) < 1e-12
    assert oracle.lib.xo_compute_scale(-1.0, 8, C.byref(out)) == 1
    assert oracle.lib.xo_compute_scale(float("inf"), 8, C.byref(out)) == 1


def test_scalar_walkthrough(oracle):
    # test_quant.cpp:27-43
    v = np.array([[1.0, 2.5, 4.0]], np.float32)
    rc, q, s = oracle.quantize(v, 8, 0, 0)
    assert rc == 0 and list(q[0]) == [31, 79, 127] and abs(s[0] - 31.75) < 1e-12
    rc, d = oracle.dequantize(q, s, 0)
    assert abs(d[0, 0] - 0.97638) < 1e-4 and abs(d[0, 1] - 2.48819) < 1e-3 and d[0, 2] == 4.0
    rc, r = oracle.residual(v, q, s, 0)
    assert abs(r[0, 0] - 0.0236) < 1e-4 and abs(r[0, 1] - 0.0118) < 1e-4 and r[0, 2] == 0.0


def test_per_row_known(oracle):
    # test_quant.cpp:54-67
    a = np.array([[1, 2], [10, 20]], np.float32)
    rc, q, s = oracle.quantize(a, 8, 1, 0)
    assert list(q.ravel()) == [63, 127, 63, 127]
    assert abs(s[0] - 63.5) < 1e-12 and abs(s[1] - 6.35) < 1e-12


def test_worked_gemm_int(oracle):
    # worked_example.hpp:42-50, test_matrix_core.cpp:47-50
    a = np.array([11, -6, 4, 3, 64, -19, -9, 6, 17], np.int8).reshape(3, 3)
    b = np.array([63, 0, -6, -5, 36, -3, -2, 0, -5], np.int8).reshape(3, 3)
    rc, p = oracle.gemm_int(a, b)
    assert p[0, 0] == 715


def test_gemm_int_overflow_guard(oracle):
    # test_matrix_core.cpp:86-97
    assert oracle.lib.xo_gemm_int_max_inner(8) == 16384
    k = 16385
    rc, _ = oracle.gemm_int(np.zeros((1, k), np.int8), np.zeros((k, 1), np.int8))
    assert rc == 1


def test_min_rule_zero_stat_row(oracle):
    # test_sparse.cpp:55-60
    a = np.array([[0.1, 0.2, 0.3], [0.1, 0.2, 0.3]], np.float32)
    rc, rp, ci, v = oracle.reduce(a, np.array([0.0, 1e6], np.float32), 1.0, 1, 10.0, True)
    assert rp[1] == 3 and rp[2] == 3


def test_quantize_csr_per_row_empty(oracle):
    # test_sparse.cpp:222-233
    rp = np.array([0, 1, 1, 2], np.int32)
    ci = np.array([0, 1], np.int32)
    v = np.array([2.0, -8.0], np.float32)
    rc, qv, s = oracle.quantize_csr(3, 3, rp, ci, v, 8, 1, 1)
    assert abs(s[0] - 63.5) < 1e-9 and s[1] == 1.0 and abs(s[2] - 127 / 8) < 1e-12
    assert list(qv) == [127, -127]


def test_splitmix_pinned(oracle):
    # test_distributions.cpp:81-89
    import ctypes as C
    st = C.c_uint64(42)
    oracle.lib.xo_splitmix_next.restype = C.c_uint64
    assert oracle.lib.xo_splitmix_next(C.byref(st)) == 13679457532755275413
    assert oracle.lib.xo_splitmix_next(C.byref(st)) == 2949826092126892291


# ---- golden vectors generated from the reference ---------------------------
def test_pipeline_golden(oracle):
    g = np.load(ol.os.path.join(GOLD, "pipeline_golden.npz"))
    n = 0
    for key in g.files:
        if not key.endswith("_meta"):
            continue
        base = key[: -len("_meta")]
        m, k, nn, sa, sb, scheme, pol, rnd, bits, path, shape = g[key]
        lo, hi, thr, s, da, db = g[base + "_fmeta"]
        a, b = g[f"shape{shape}_a"], g[f"shape{shape}_b"]
        c = ol.cfg(bits=int(bits), threshold=thr, density_limit=s, scheme=int(scheme),
                   policy=int(pol), rounding=int(rnd))
        rc, out, rep = oracle.xigemm(a, b, config=c)
        assert rc == 0
        assert bits_eq(out, g[base + "_xigemm"]), base
        assert rep.path == path and rep.density_a == da and rep.density_b == db
        rc, full, _ = oracle.xigemm(a, b, config=c, reduce=False)
        assert bits_eq(full, g[base + "_full"]), base
        rc, direct = oracle.gemm_direct(a, b, config=c)
        assert bits_eq(direct, g[base + "_direct"]), base
        n += 1
    assert n == 49


def test_stage_golden(oracle):
    g = np.load(ol.os.path.join(GOLD, "stages_golden.npz"))
    pres = sorted({k.split("cfg")[0] for k in g.files if k.endswith("cfg")})
    for pre in pres:
        thr, s, scheme, pol, rnd, bits = g[pre + "cfg"]
        c = ol.cfg(bits=int(bits), threshold=thr, density_limit=s, scheme=int(scheme),
                   policy=int(pol), rounding=int(rnd))
        rc, d = oracle.dump(g[pre + "a"], g[pre + "b"], c)
        assert rc == 0
        for name in d:
            if name == "result":
                continue
            assert bits_eq(d[name], g[pre + name]), (pre, name)


def test_known_answers_golden(oracle):
    g = np.load(ol.os.path.join(GOLD, "known_answers.npz"))
    for bits in (4, 8):
        for rnd in (0, 1):
            for scheme in (0, 1, 2):
                pre = f"q_{bits}_{rnd}_{scheme}_"
                rc, q, s = oracle.quantize(g[pre + "in"], bits, scheme, rnd)
                assert bits_eq(q, g[pre + "q"]) and bits_eq(s, g[pre + "s"])
    x = np.array([[1.0, -2.0, 3.0e-3, 0.0]], np.float32)
    for rnd in (0, 1):
        rc, q = oracle.quantize_with_scales(x, np.array([1e300]), 8, 0, rnd)
        assert bits_eq(q, g[f"huge_{rnd}"])


# ---- live comparison against the reference build ----------------------------
@pytest.mark.parametrize("seed", range(12))
def test_pipeline_vs_ref_random(oracle, ref, seed):
    rng = np.random.default_rng(seed)
    m, k, n = (int(x) for x in rng.integers(1, 70, size=3))
    a = ol.random_dense(m, k, seed * 2 + 1, -3, 3)
    b = ol.random_dense(k, n, seed * 2 + 2, -3, 3)
    for scheme in (0, 1):
        for pol in (0, 1):
            thr = float(10 ** rng.uniform(-3, 0.5))
            c = ol.cfg(bits=int(rng.choice([4, 8])), threshold=thr,
                       density_limit=float(rng.uniform(0.05, 1.0)), scheme=scheme, policy=pol,
                       rounding=int(rng.integers(0, 2)))
            cm = ol.random_dense(m, n, seed + 99, -1, 1)
            r1 = oracle.xigemm(a, b, c=cm, alpha=1.5, beta=-0.25, config=c)
            r2 = ref.xigemm(a, b, c=cm, alpha=1.5, beta=-0.25, config=c)
            assert r1[0] == r2[0] == 0
            assert bits_eq(r1[1], r2[1])
            assert (r1[2].density_a, r1[2].density_b, r1[2].path) == \
                   (r2[2].density_a, r2[2].density_b, r2[2].path)


def test_stage_functions_vs_ref(oracle, ref):
    a = ol.random_dense(17, 23, 5, -7, 7)
    for bits in (4, 8):
        for rnd in (0, 1):
            for scheme in (0, 1, 2):
                r1, r2 = oracle.quantize(a, bits, scheme, rnd), ref.quantize(a, bits, scheme, rnd)
                assert bits_eq(r1[1], r2[1]) and bits_eq(r1[2], r2[2])
                assert bits_eq(oracle.dequantize(r1[1], r1[2], scheme)[1],
                               ref.dequantize(r2[1], r2[2], scheme)[1])
                assert bits_eq(oracle.residual(a, r1[1], r1[2], scheme)[1],
                               ref.residual(a, r2[1], r2[2], scheme)[1])
    d = ol.random_dense(19, 11, 8, -4, 4)
    for f in ("avg_vectors", "abs_min_vectors"):
        x, y = getattr(oracle, f)(d), getattr(ref, f)(d)
        assert bits_eq(x[1], y[1]) and bits_eq(x[2], y[2])
    for per_row in (True, False):
        for pol in (0, 1):
            st = np.abs(ol.random_dense(19 if per_row else 11, 1, 3, 0, 2)).ravel()
            x = oracle.reduce(d, st, 0.7, pol, 3.0, per_row)
            y = ref.reduce(d, st, 0.7, pol, 3.0, per_row)
            for u, v in zip(x[1:], y[1:]):
                assert bits_eq(u, v)
            for scheme in (0, 1, 2):
                qa = oracle.quantize_csr(19, 11, x[1], x[2], x[3], 8, scheme, 1)
                qb = ref.quantize_csr(19, 11, y[1], y[2], y[3], 8, scheme, 1)
                assert bits_eq(qa[1], qb[1]) and bits_eq(qa[2], qb[2])
            dq = np.clip(np.round(ol.random_dense(11, 9, 4, -127, 127)), -127, 127).astype(np.int8)
            assert bits_eq(oracle.spmm_int(19, 11, x[1], x[2], qa[1], dq)[1],
                           ref.spmm_int(19, 11, y[1], y[2], qb[1], dq)[1])
            df = ol.random_dense(11, 9, 5, -2, 2)
            assert bits_eq(oracle.spmm_f32(19, 11, x[1], x[2], x[3], df)[1],
                           ref.spmm_f32(19, 11, y[1], y[2], y[3], df)[1])
            t1 = oracle.csr_transpose_i8(19, 11, x[1], x[2], qa[1])
            t2 = ref.csr_transpose_i8(19, 11, y[1], y[2], qb[1])
            for u, v in zip(t1[1:], t2[1:]):
                assert bits_eq(u, v)
    x = ol.random_dense(13, 17, 9, -3, 3)
    y = ol.random_dense(17, 6, 10, -3, 3)
    assert bits_eq(oracle.gemm_f32(x, y)[1], ref.gemm_f32(x, y)[1])
    cc = ol.random_dense(13, 6, 11, -3, 3)
    dd = ol.random_dense(13, 6, 12, -3, 3)
    assert bits_eq(oracle.axpby(dd, 2.0, cc, -0.5)[1], ref.axpby(dd, 2.0, cc, -0.5)[1])
    for kind, p1, p2 in ((0, 0, 0), (1, 10.0, 3.0), (2, 1.5, 0), (3, 4.0, 0), (4, 3, 0)):
        assert bits_eq(oracle.generate(kind, p1, p2, 42, 8, 9)[1], ref.generate(kind, p1, p2, 42, 8, 9)[1])


# ---- the restatement against the reference at the sizes the GPU parity tests use
def _student_t(rows, cols, seed):
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((rows, cols))
    chi = (rng.standard_normal((3, rows, cols)) ** 2).sum(0) / 3.0
    return (z / np.sqrt(chi)).astype(np.float32)


@pytest.mark.parametrize("shape,data,scheme,pol,thr", [
    ((1024, 1024, 1024), "uniform", 1, 0, 0.112),    # C1: VectorWise AvgRule, ~5% kept
    ((1024, 1024, 1024), "uniform", 0, 1, 0.5),      # reference defaults (PerTensor, MinRule)
    ((1280, 2048, 1152), "t3", 1, 0, 0.02),           # heavy-tailed, K = 2048, ragged M / N
])
def test_restatement_vs_ref_large(oracle, ref, shape, data, scheme, pol, thr):
    """oracle/xigemm_oracle.c against the unmodified reference (oracle/_ref) at
    >= 1024 per dimension: every stage intermediate of the pipeline dump and the
    final C, bit for bit (the large-shape GPU parity tests use these stage
    functions as their checker)."""
    m, k, n = shape
    if data == "uniform":
        a = ol.random_dense(m, k, 1, -1, 1)
        b = ol.random_dense(k, n, 2, -1, 1)
    else:
        a, b = _student_t(m, k, 1), _student_t(k, n, 2)
    c = ol.cfg(bits=8, threshold=thr, density_limit=0.3, scheme=scheme, policy=pol, rounding=1)
    rc1, d1 = oracle.dump(a, b, c)
    rc2, d2 = ref.dump(a, b, c)
    assert rc1 == rc2 == 0
    for name in d1:
        if name == "result" or name not in d2:
            continue
        assert bits_eq(d1[name], d2[name]), name
    r1 = oracle.xigemm(a, b, config=c)
    r2 = ref.xigemm(a, b, config=c)
    assert bits_eq(r1[1], r2[1])
    assert (r1[2].density_a, r1[2].density_b, r1[2].path) == (r2[2].density_a, r2[2].density_b, r2[2].path)
    assert max(r1[2].density_a, r1[2].density_b) > 0.0
