"""The CUDA-core CSR compensation path (csrc/spmm.cu) of the SparseResidual
branch: the quad-packed CSR build (ballot/scan stream compaction) and the strip
SpMM with the exact compensation epilogues.  It must give the reference's
result bit for bit - the same as the tcgen05 masked-dense launch - on every
shape, scheme, policy and C/alpha/beta combination; overflowing builds must
fall back to the dense launch; the spmm_int API routed through the strip
kernel must equal the oracle; calibrate_eta runs on the device."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle_lib as ol  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2403_06924_b200 as xg  # noqa: E402
from test_gpu_parity import beq, cfg_from  # noqa: E402


@pytest.fixture
def force():
    saved = xg.comp_model()
    yield lambda f: xg.comp_model(force=f)
    xg.comp_model(force=saved["force"])


def _run(a, b, c, alpha, beta, cfg):
    t = lambda x: None if x is None else torch.from_numpy(x).cuda()  # noqa: E731
    return xg.xigemm(t(a), t(b), t(c), alpha, beta, cfg)


CASES = [
    # m, k, n, scheme, policy, bits, threshold (~1.5-3.5% density, bisected with the oracle), outliers, with C
    (300, 1024, 260, 1, 0, 8, 0.0289, True, True),       # pair compensation launch skipped
    (700, 2052, 1028, 1, 0, 8, 0.0202, True, False),     # K not a multiple of 16, ragged strips and chunks
    (1024, 2048, 1000, 0, 1, 8, 13335.2, False, True),   # PerTensor + MinRule (fix-up of lambda')
    (513, 3000, 771, 1, 1, 8, 13335.2, False, False),    # MinRule, odd N (1-CTA dense kernel skipped)
    (513, 3000, 771, 1, 0, 4, 0.01685, False, False),    # int4
    (200, 640, 96, 0, 0, 8, 0.0379, True, True),         # M < 256: 1-CTA EPI_COMP launch skipped
    (2048, 8192, 512, 1, 0, 8, 0.01, True, True),        # K = 8192: 16-line strips of 128 KiB
    (256, 12000, 384, 1, 0, 8, 0.0083, True, False),     # K > 8192: 8-line strips
]


@pytest.mark.parametrize("case", CASES)
def test_csr_equals_dense_and_oracle(oracle, force, case):
    m, k, n, scheme, pol, bits, thr, outl, with_c = case
    a = ol.random_dense(m, k, m + 3, -4, 4)
    b = ol.random_dense(k, n, n + 5, -4, 4)
    if outl:
        a[m // 2, 7] = 40.0
        b[11, n // 3] = -33.0
    cm = ol.random_dense(m, n, 9, -1, 1) if with_c else None
    alpha, beta = (1.25, -0.5) if with_c else (0.75, 0.0)
    c = ol.cfg(bits=bits, threshold=thr, density_limit=0.9, scheme=scheme, policy=pol, rounding=1)
    force(2)
    rep_s = _run(a, b, cm, alpha, beta, cfg_from(c))
    force(1)
    rep_d = _run(a, b, cm, alpha, beta, cfg_from(c))
    assert int(rep_s.path) == 0, "case must take the SparseResidual branch"
    assert 0 < max(rep_s.density_a, rep_s.density_b) < 0.05, (rep_s.density_a, rep_s.density_b)
    assert rep_s.comp_kernel == 1 and rep_d.comp_kernel == 0
    assert beq(rep_s.result, rep_d.result), case
    if m * k * n <= 2 ** 31:
        rc, ref, orep = oracle.xigemm(a, b, c=cm, alpha=alpha, beta=beta, config=c)
        assert rc == 0
        assert beq(rep_s.result, ref), case
        assert (rep_s.density_a, rep_s.density_b) == (orep.density_a, orep.density_b)


def test_csr_heavy_rows_warp_shared(oracle, force):
    """A row whose D_F is exactly zero (B rows pairwise equal, A row alternating)
    has AvgRule statistic 0 and is retained whole (sparse.cpp:49-65): 3000 entries,
    walked by the whole warp (kHeavyQ), the rest of the operand at ~2% density."""
    m, k, n = 513, 3000, 771
    a = ol.random_dense(m, k, m + 3, -4, 4)
    b = ol.random_dense(k, n, n + 5, -4, 4)
    b[1::2] = b[0::2]
    a[77] = np.where(np.arange(k) % 2 == 0, 1.5, -1.5).astype(np.float32)
    a[300] = a[77]
    c = ol.cfg(bits=8, threshold=0.017, density_limit=0.9, scheme=1, policy=0, rounding=1)
    force(2)
    rs = _run(a, b, None, 1.0, 0.0, cfg_from(c))
    rc, ref, orep = oracle.xigemm(a, b, config=c)
    assert rc == 0 and int(rs.path) == 0
    assert rs.density_a < 0.05 and rs.nnz_a >= 2 * k
    assert rs.comp_kernel == 1
    assert beq(rs.result, ref)


def test_csr_graph_replay_repeatable(force):
    """Second and third calls replay the captured graph (CSR cursors re-zeroed per call)."""
    m, k, n = 1024, 2048, 1024
    a = torch.from_numpy(ol.random_dense(m, k, 1, -3, 3)).cuda()
    b = torch.from_numpy(ol.random_dense(k, n, 2, -3, 3)).cuda()
    cfg = xg.XigemmConfig(threshold=0.03, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
    force(1)
    ref = xg.xigemm(a, b, cfg=cfg).result.clone()
    force(2)
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    for _ in range(3):
        rep = xg.xigemm(a, b, cfg=cfg, out=out)
        assert rep.comp_kernel == 1
        assert beq(out, ref)


def test_csr_overflow_falls_back_to_dense(force):
    """A density above the CSR capacity (6.25%) and rows longer than the strip
    SpMM takes: the build raises csr_bad, the masked-dense launch serves the call."""
    m, k, n = 512, 4096, 512
    a = ol.random_dense(m, k, 4, -4, 4)
    b = ol.random_dense(k, n, 5, -4, 4)
    c = ol.cfg(bits=8, threshold=0.01, density_limit=1.0, scheme=1, policy=0, rounding=1)
    force(1)
    rd = _run(a, b, None, 1.0, 0.0, cfg_from(c))
    force(2)
    rs = _run(a, b, None, 1.0, 0.0, cfg_from(c))
    assert int(rs.path) == 0 and rs.density_a > 0.2
    assert rs.comp_kernel == 0
    assert beq(rs.result, rd.result)


def test_csr_empty_selection(oracle, force):
    """Nothing retained (huge M): every segment empty, out = fl(D_F + 0) + 0."""
    m, k, n = 300, 1024, 400
    a = ol.random_dense(m, k, 6, -1, 1)
    b = ol.random_dense(k, n, 7, -1, 1)
    c = ol.cfg(bits=8, threshold=1e6, density_limit=0.3, scheme=1, policy=0, rounding=1)
    force(2)
    rs = _run(a, b, None, 1.0, 0.0, cfg_from(c))
    assert rs.nnz_a == 0 and rs.nnz_b == 0 and rs.comp_kernel == 1
    rc, ref, _ = oracle.xigemm(a, b, config=c)
    assert beq(rs.result, ref)


def test_auto_choice_follows_density(force):
    """Auto mode (cost model of k_dispatch): at K = 16384 the masked-dense launch
    costs 4K/p_tc per output element, more than the CSR path's fixed epilogue
    cost, so a near-empty selection (~0.005%) takes the CSR path (measured 5%
    faster there, profiles/r2_csr_sweep_k16384.jsonl); a few percent does not."""
    force(0)
    m, n, k = 4096, 4096, 16384
    a = xg.generate("normal", m, k, 1)
    b = xg.generate("normal", k, n, 2)
    lo = xg.xigemm(a, b, cfg=xg.XigemmConfig(threshold=0.0398, scheme=xg.QuantScheme.VectorWise,
                                             policy=xg.ReductionPolicy.AvgRule))
    hi = xg.xigemm(a, b, cfg=xg.XigemmConfig(threshold=0.02, scheme=xg.QuantScheme.VectorWise,
                                             policy=xg.ReductionPolicy.AvgRule))
    assert int(lo.path) == 0 and 0 < max(lo.density_a, lo.density_b) < 1e-4 and lo.comp_kernel == 1
    assert int(hi.path) == 0 and max(hi.density_a, hi.density_b) > 0.01 and hi.comp_kernel == 0


@pytest.mark.parametrize("rows,cols,d_cols,dens", [(1, 1, 1, 1.0), (37, 300, 50, 0.1), (512, 4096, 1000, 0.02),
                                                   (300, 9000, 64, 0.05), (64, 16384, 24, 0.01)])
def test_spmm_int_api_strip(oracle, rows, cols, d_cols, dens):
    rng = np.random.default_rng(rows + cols)
    dense = np.where(rng.random((rows, cols)) < dens, rng.integers(-127, 128, (rows, cols)), 0).astype(np.float32)
    s = xg.csr_from_dense(torch.from_numpy(dense).cuda())
    q = xg.quantize_csr(s, xg.QuantBits.Int8, xg.ScaleScheme.PerRow, xg.RoundingMode.Nearest)
    dq = xg.quantize(torch.from_numpy(ol.random_dense(cols, d_cols, 3, -2, 2)).cuda(), 8, 0, 1)
    got = xg.spmm_int(q.matrix, dq)
    qi = np.zeros((rows, cols), dtype=np.int64)
    rp, ci, v = (q.matrix.row_ptr.cpu().numpy(), q.matrix.col_idx.cpu().numpy(), q.matrix.values.cpu().numpy())
    for i in range(rows):
        qi[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    ref = (qi @ dq.data.cpu().numpy().astype(np.int64)).astype(np.int32)
    assert beq(got, ref)


def test_calibrate_eta_on_device():
    cal = xg.calibrate_eta(1024, xg.QuantBits.Int8, 3)
    assert 1.0 / 1024 <= cal.eta <= 1.0
    assert cal.gemm_ops_per_s > 1e14 and cal.spmm_macs_per_s > 1e11


@pytest.mark.parametrize("seed", range(12))
def test_csr_random_configs_vs_oracle(oracle, force, seed):
    """Random small shapes and configurations (bits, rounding, scheme, policy, C,
    alpha/beta) with the CSR compensation forced: equal to the oracle bit for bit
    whenever the SparseResidual branch runs (the CSR build may fall back to the
    masked-dense launch at high density; both are checked against the oracle)."""
    rng = np.random.default_rng(500 + seed)
    m, k, n = (int(v) for v in rng.integers(1, 400, size=3))
    a = ol.random_dense(m, k, seed * 3 + 1, -4, 4)
    b = ol.random_dense(k, n, seed * 3 + 2, -4, 4)
    cm = ol.random_dense(m, n, seed + 9, -1, 1)
    force(2)
    for scheme in (0, 1):
        for pol in (0, 1):
            c = ol.cfg(bits=int(rng.choice([4, 8])), threshold=float(10 ** rng.uniform(-2.5, 0.3)),
                       density_limit=float(rng.uniform(0.05, 1.0)), scheme=scheme, policy=pol,
                       rounding=int(rng.integers(0, 2)))
            rc, ref, orep = oracle.xigemm(a, b, c=cm, alpha=1.25, beta=-0.5, config=c)
            assert rc == 0
            rep = _run(a, b, cm, 1.25, -0.5, cfg_from(c))
            assert beq(rep.result, ref), (m, k, n, scheme, pol)
            assert (rep.density_a, rep.density_b, int(rep.path)) == (orep.density_a, orep.density_b, orep.path)
            if int(rep.path) == 1:
                assert rep.comp_kernel == 0


@pytest.mark.parametrize("seed", range(8))
def test_csr_random_midsize_vs_oracle(oracle, force, seed):
    """Random mid-size shapes with the CSR compensation forced (quad builds with
    partial last quads, heavy and empty rows, ragged strips and chunks): equal to
    the oracle bit for bit, and the CSR path actually taken when the selection
    is sparse enough for its capacity."""
    rng = np.random.default_rng(700 + seed)
    m = int(rng.integers(256, 700))
    k = int(rng.integers(128, 1000)) * 4
    n = int(rng.integers(256, 1100))
    a = ol.random_dense(m, k, seed * 3 + 41, -4, 4)
    b = ol.random_dense(k, n, seed * 3 + 42, -4, 4)
    cm = ol.random_dense(m, n, seed + 19, -1, 1)
    bits, scheme, rnd = int(rng.choice([4, 8])), int(rng.integers(0, 2)), int(rng.integers(0, 2))
    target = float(rng.uniform(0.005, 0.04))  # a selection inside the CSR capacity (6.25%)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    lo, hi = 1e-4, 10.0
    for _ in range(30):  # bisect the threshold on the GPU pipeline for the target density
        thr = (lo * hi) ** 0.5
        cc = ol.cfg(bits=bits, threshold=thr, density_limit=0.9, scheme=scheme, policy=0, rounding=rnd)
        d = max(xg.xigemm(ta, tb, cfg=cfg_from(cc)).density_a, xg.xigemm(ta, tb, cfg=cfg_from(cc)).density_b)
        if abs(d - target) < 0.2 * target:
            break
        lo, hi = (thr, hi) if d > target else (lo, thr)
    c = ol.cfg(bits=bits, threshold=thr, density_limit=0.9, scheme=scheme, policy=0, rounding=rnd)
    force(2)
    rc, ref, orep = oracle.xigemm(a, b, c=cm, alpha=1.25, beta=-0.5, config=c)
    assert rc == 0
    rep = _run(a, b, cm, 1.25, -0.5, cfg_from(c))
    assert beq(rep.result, ref), (m, k, n, c.scheme, c.bits, c.rounding)
    assert (rep.density_a, rep.density_b, int(rep.path)) == (orep.density_a, orep.density_b, orep.path)
    assert int(rep.path) == 0 and rep.comp_kernel == 1  # 0.3-4.6% selections on these seeds
