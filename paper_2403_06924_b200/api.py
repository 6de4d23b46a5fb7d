"""Python mirror of the reference's public API (proj/include/xigemm/*.hpp),
executed by the sm_100a kernels through the C-ABI.

Names, argument meaning, defaults and error behaviour follow the reference:
validation failures raise `InvalidArgument` (a ValueError) exactly where the
reference throws std::invalid_argument.  Matrices are torch tensors on the
CUDA device (device memory / streams are plumbing provided by PyTorch); numpy
arrays are accepted and copied to the device (results then come back as numpy).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import DUMP_FIELDS, InvalidArgument, XgConfig, XgDump, XgReport, check, lib


# ---- enums (reference declaration order) -----------------------------------
class QuantBits(enum.IntEnum):      # quantize.hpp:12
    Int4 = 4
    Int8 = 8


class RoundingMode(enum.IntEnum):   # quantize.hpp:18
    Floor = 0
    Nearest = 1


class ScaleScheme(enum.IntEnum):    # quantize.hpp:20
    PerTensor = 0
    PerRow = 1
    PerColumn = 2


class QuantScheme(enum.IntEnum):    # pipeline.hpp:15
    PerTensor = 0
    VectorWise = 1


class ReductionPolicy(enum.IntEnum):  # sparse.hpp:40
    AvgRule = 0
    MinRule = 1


class GemmPath(enum.IntEnum):       # pipeline.hpp:30
    SparseResidual = 0
    DenseResidual = 1


def quant_max(bits) -> int:         # quantize.hpp:16
    return (1 << (int(bits) - 1)) - 1


def gemm_int_max_inner(bits) -> int:  # quantize.hpp:103
    return int(lib().xg_gemm_max_inner(int(bits)))


@dataclass
class XigemmConfig:                 # pipeline.hpp:19-28
    bits: QuantBits = QuantBits.Int8
    threshold: float = 0.5
    density_limit: float = 0.3
    scheme: QuantScheme = QuantScheme.PerTensor
    policy: ReductionPolicy = ReductionPolicy.MinRule
    rounding: RoundingMode = RoundingMode.Nearest

    def c(self) -> XgConfig:
        return XgConfig(int(self.bits), float(self.threshold), float(self.density_limit),
                        int(self.scheme), int(self.policy), int(self.rounding))

    def validate(self) -> None:     # pipeline.cpp:153-160
        if not self.threshold > 0.0:
            raise InvalidArgument("XigemmConfig: threshold M must be positive")
        if not self.density_limit > 0.0 or self.density_limit > 1.0:
            raise InvalidArgument("XigemmConfig: density limit must be in (0, 1]")


@dataclass
class ScaleFactors:                 # quantize.hpp:24-46
    scheme: ScaleScheme = ScaleScheme.PerTensor
    values: torch.Tensor = None     # float64 on device


@dataclass
class QuantizedMatrix:              # quantize.hpp:50-69
    rows: int
    cols: int
    data: torch.Tensor              # int8 rows x cols
    bits: QuantBits
    scales: ScaleFactors
    rounding: RoundingMode


@dataclass
class SparseCsr:                    # sparse.hpp:14-32
    rows: int
    cols: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    values: torch.Tensor

    def nnz(self) -> int:
        return int(self.values.numel())


@dataclass
class QuantizedCsr:                 # sparse.hpp:34-38
    matrix: SparseCsr
    bits: QuantBits
    scales: ScaleFactors


@dataclass
class GemmReport:                   # pipeline.hpp:32-39
    result: torch.Tensor
    density_a: float = 0.0
    density_b: float = 0.0
    path: GemmPath = GemmPath.DenseResidual
    timings: dict = field(default_factory=dict)
    nnz_a: int = 0
    nnz_b: int = 0
    stats_fallbacks: int = 0
    comp_kernel: int = 0            # sparse terms ran on 0: tcgen05 masked-dense, 1: CUDA-core CSR SpMM


# ---- plumbing -----------------------------------------------------------------
def _dev(x, dtype) -> tuple[torch.Tensor, bool]:
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype), True
    if x.device.type != "cuda":
        return x.to("cuda", dtype).contiguous(), True
    return x.to(dtype).contiguous(), False


def _ret(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t


def _p(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _s() -> C.c_void_p:
    # the raw handle of the current stream without building a torch Stream object
    # (a few microseconds per call on the pipeline's latency-bound host path)
    return C.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


def _nscales(scheme, rows, cols) -> int:
    return rows if scheme == ScaleScheme.PerRow else cols if scheme == ScaleScheme.PerColumn else 1


def _scales_dev(s: ScaleFactors) -> torch.Tensor:
    v = s.values
    if isinstance(v, (list, tuple)):
        v = torch.tensor(v, dtype=torch.float64)
    if isinstance(v, np.ndarray):
        v = torch.from_numpy(v)
    return v.to("cuda", torch.float64).contiguous()


def _validate_scales(s: ScaleFactors, rows, cols):    # quantize.cpp:44-56
    v = _scales_dev(s)
    if v.numel() != _nscales(s.scheme, rows, cols):
        raise InvalidArgument("ScaleFactors: value count does not match scheme")
    return v


# ---- quantize.hpp ---------------------------------------------------------
def compute_scale(max_abs: float, bits) -> float:     # quantize.cpp:99-105
    if not (max_abs >= 0.0) or not np.isfinite(max_abs):
        raise InvalidArgument("compute_scale: max_abs must be finite and nonnegative")
    return 1.0 if max_abs == 0.0 else float(quant_max(bits)) / float(max_abs)


def quantize(a, bits=QuantBits.Int8, scheme=ScaleScheme.PerTensor,
             rounding=RoundingMode.Nearest) -> QuantizedMatrix:
    x, host = _dev(a, torch.float32)
    rows, cols = x.shape
    q = torch.empty((rows, cols), dtype=torch.int8, device="cuda")
    sc = torch.empty(_nscales(scheme, rows, cols), dtype=torch.float64, device="cuda")
    check(lib().xg_quantize(_p(x), rows, cols, int(bits), int(scheme), int(rounding), _p(q),
                            _p(sc), _s()))
    return QuantizedMatrix(rows, cols, q, QuantBits(int(bits)), ScaleFactors(ScaleScheme(int(scheme)), sc),
                           RoundingMode(int(rounding)))


def quantize_with_scales(a, bits, scales: ScaleFactors, rounding) -> QuantizedMatrix:
    x, _ = _dev(a, torch.float32)
    rows, cols = x.shape
    sv = _validate_scales(scales, rows, cols)
    q = torch.empty((rows, cols), dtype=torch.int8, device="cuda")
    check(lib().xg_quantize_with_scales(_p(x), rows, cols, int(bits), int(scales.scheme), _p(sv),
                                        int(rounding), _p(q), _s()))
    return QuantizedMatrix(rows, cols, q, QuantBits(int(bits)), ScaleFactors(scales.scheme, sv),
                           RoundingMode(int(rounding)))


def dequantize(q: QuantizedMatrix) -> torch.Tensor:
    out = torch.empty((q.rows, q.cols), dtype=torch.float32, device="cuda")
    check(lib().xg_dequantize(_p(q.data), q.rows, q.cols, int(q.scales.scheme),
                              _p(_scales_dev(q.scales)), _p(out), _s()))
    return out


def residual(a, q: QuantizedMatrix) -> torch.Tensor:
    x, _ = _dev(a, torch.float32)
    if tuple(x.shape) != (q.rows, q.cols):
        raise InvalidArgument("residual: shape mismatch")
    out = torch.empty_like(x)
    check(lib().xg_residual(_p(x), _p(q.data), q.rows, q.cols, int(q.scales.scheme),
                            _p(_scales_dev(q.scales)), _p(out), _s()))
    return out


def dequant_product(p, scales_a: ScaleFactors, scales_b: ScaleFactors) -> torch.Tensor:
    x, _ = _dev(p, torch.int32)
    rows, cols = x.shape
    if scales_a.scheme == ScaleScheme.PerColumn:
        raise InvalidArgument("dequant_product: left scales must be PerTensor or PerRow")
    if scales_b.scheme == ScaleScheme.PerRow:
        raise InvalidArgument("dequant_product: right scales must be PerTensor or PerColumn")
    sa = _validate_scales(scales_a, rows, 1)
    sb = _validate_scales(scales_b, 1, cols)
    out = torch.empty((rows, cols), dtype=torch.float32, device="cuda")
    check(lib().xg_dequant_product(_p(x), rows, cols, int(scales_a.scheme), _p(sa),
                                   int(scales_b.scheme), _p(sb), _p(out), _s()))
    return out


def gemm_int(a: QuantizedMatrix, b: QuantizedMatrix) -> torch.Tensor:
    if a.cols != b.rows:
        raise InvalidArgument("gemm_int: inner dimensions do not match")
    out = torch.empty((a.rows, b.cols), dtype=torch.int32, device="cuda")
    check(lib().xg_gemm_i8(_p(a.data), _p(b.data), a.rows, a.cols, b.cols, int(a.bits),
                           int(b.bits), _p(out), _s()))
    return out


def gemm_i8(a, b, bits_a=8, bits_b=8) -> torch.Tensor:
    """Raw int8 x int8 -> int32 product of row-major device tensors."""
    x, _ = _dev(a, torch.int8)
    y, _ = _dev(b, torch.int8)
    if x.shape[1] != y.shape[0]:
        raise InvalidArgument("gemm_int: inner dimensions do not match")
    out = torch.empty((x.shape[0], y.shape[1]), dtype=torch.int32, device="cuda")
    check(lib().xg_gemm_i8(_p(x), _p(y), x.shape[0], x.shape[1], y.shape[1], bits_a, bits_b,
                           _p(out), _s()))
    return out


# ---- matrix.hpp -----------------------------------------------------------
def gemm_f32(a, b):
    x, host = _dev(a, torch.float32)
    y, _ = _dev(b, torch.float32)
    if x.shape[1] != y.shape[0]:
        raise InvalidArgument("gemm_f32: inner dimensions do not match")
    out = torch.empty((x.shape[0], y.shape[1]), dtype=torch.float32, device="cuda")
    check(lib().xg_gemm_f32(_p(x), _p(y), x.shape[0], x.shape[1], y.shape[1], _p(out), _s()))
    return _ret(out, host)


def axpby_inplace(d: torch.Tensor, alpha: float, c, beta: float) -> torch.Tensor:
    y, _ = _dev(c, torch.float32)
    if tuple(d.shape) != tuple(y.shape):
        raise InvalidArgument("axpby_inplace: shape mismatch")
    check(lib().xg_axpby(_p(d), float(alpha), _p(y), float(beta), d.numel(), _s()))
    return d


def subtract(a, b):
    x, host = _dev(a, torch.float32)
    y, _ = _dev(b, torch.float32)
    if x.shape != y.shape:
        raise InvalidArgument("subtract: shape mismatch")
    out = torch.empty_like(x)
    check(lib().xg_subtract(_p(x), _p(y), _p(out), x.numel(), _s()))
    return _ret(out, host)


def add_inplace(d: torch.Tensor, x) -> torch.Tensor:
    y, _ = _dev(x, torch.float32)
    if d.shape != y.shape:
        raise InvalidArgument("add_inplace: shape mismatch")
    check(lib().xg_add_inplace(_p(d), _p(y), d.numel(), _s()))
    return d


def max_abs_finite(a) -> tuple[float, bool]:
    x, _ = _dev(a, torch.float32)
    m = C.c_float(0)
    f = C.c_int(0)
    check(lib().xg_max_abs(_p(x), x.numel(), C.byref(m), C.byref(f), _s()))
    return m.value, bool(f.value)


# ---- sparse.hpp -------------------------------------------------------------
def _reduce(m, stat, thr, policy, scale_other, per_row) -> SparseCsr:
    x, _ = _dev(m, torch.float32)
    rows, cols = x.shape
    st, _ = _dev(stat if not isinstance(stat, list) else np.asarray(stat, np.float32), torch.float32)
    if st.numel() != (rows if per_row else cols):
        raise InvalidArgument("reduce: stat vector length mismatch")
    rp = torch.empty(rows + 1, dtype=torch.int32, device="cuda")
    nnz = C.c_int64(0)
    L = lib()
    check(L.xg_reduce_count(_p(x), rows, cols, _p(st), float(thr), int(policy), float(scale_other),
                            int(per_row), _p(rp), C.byref(nnz), _s()))
    ci = torch.empty(max(1, nnz.value), dtype=torch.int32, device="cuda")
    v = torch.empty(max(1, nnz.value), dtype=torch.float32, device="cuda")
    check(L.xg_reduce_fill(_p(x), rows, cols, _p(st), float(thr), int(policy), float(scale_other),
                           int(per_row), _p(rp), _p(ci), _p(v), _s()))
    return SparseCsr(rows, cols, rp, ci[: nnz.value], v[: nnz.value])


def reduce_a(a, c_row_stat, m, policy, scale_other=1.0) -> SparseCsr:   # sparse.hpp:46
    return _reduce(a, c_row_stat, m, policy, scale_other, True)


def reduce_b(b, c_col_stat, m, policy, scale_other=1.0) -> SparseCsr:   # sparse.hpp:52
    return _reduce(b, c_col_stat, m, policy, scale_other, False)


def density(s: SparseCsr) -> float:                                      # sparse.cpp:87-95
    if s.rows == 0 or s.cols == 0:
        return 0.0
    return float(s.nnz()) / (float(s.rows) * s.cols)


def csr_from_dense(a) -> SparseCsr:
    x, _ = _dev(a, torch.float32)
    rows, cols = x.shape
    rp = torch.empty(rows + 1, dtype=torch.int32, device="cuda")
    nnz = C.c_int64(0)
    check(lib().xg_csr_from_dense_count(_p(x), rows, cols, _p(rp), C.byref(nnz), _s()))
    ci = torch.empty(max(1, nnz.value), dtype=torch.int32, device="cuda")
    v = torch.empty(max(1, nnz.value), dtype=torch.float32, device="cuda")
    check(lib().xg_csr_from_dense_fill(_p(x), rows, cols, _p(rp), _p(ci), _p(v), _s()))
    return SparseCsr(rows, cols, rp, ci[: nnz.value], v[: nnz.value])


def densify(s: SparseCsr) -> torch.Tensor:
    out = torch.empty((s.rows, s.cols), dtype=torch.float32, device="cuda")
    check(lib().xg_densify(s.rows, s.cols, _p(s.row_ptr), _p(s.col_idx), _p(s.values), _p(out),
                           _s()))
    return out


def quantize_csr(s: SparseCsr, bits, scheme, rounding) -> QuantizedCsr:
    qv = torch.empty(max(1, s.nnz()), dtype=torch.int8, device="cuda")
    sc = torch.empty(_nscales(scheme, s.rows, s.cols), dtype=torch.float64, device="cuda")
    check(lib().xg_quantize_csr(s.rows, s.cols, _p(s.row_ptr), _p(s.col_idx), _p(s.values),
                                s.nnz(), int(bits), int(scheme), int(rounding), _p(qv), _p(sc),
                                _s()))
    m = SparseCsr(s.rows, s.cols, s.row_ptr, s.col_idx, qv[: s.nnz()])
    return QuantizedCsr(m, QuantBits(int(bits)), ScaleFactors(ScaleScheme(int(scheme)), sc))


def csr_transpose(s: SparseCsr) -> SparseCsr:
    nnz = s.nnz()
    trp = torch.empty(s.cols + 1, dtype=torch.int32, device="cuda")
    tci = torch.empty(max(1, nnz), dtype=torch.int32, device="cuda")
    tv = torch.empty(max(1, nnz), dtype=s.values.dtype, device="cuda")
    f = lib().xg_csr_transpose_i8 if s.values.dtype == torch.int8 else lib().xg_csr_transpose_f32
    check(f(s.rows, s.cols, _p(s.row_ptr), _p(s.col_idx), _p(s.values), nnz, _p(trp), _p(tci),
            _p(tv), _s()))
    return SparseCsr(s.cols, s.rows, trp, tci[:nnz], tv[:nnz])


def spmm_int(s: SparseCsr, d: QuantizedMatrix) -> torch.Tensor:
    if s.cols != d.rows:
        raise InvalidArgument("spmm_int: inner dimensions do not match")
    out = torch.empty((s.rows, d.cols), dtype=torch.int32, device="cuda")
    check(lib().xg_spmm_i8(s.rows, s.cols, _p(s.row_ptr), _p(s.col_idx), _p(s.values),
                           _p(d.data), d.cols, int(d.bits), _p(out), _s()))
    return out


def spmm(s: SparseCsr, d) -> torch.Tensor:
    y, _ = _dev(d, torch.float32)
    if s.cols != y.shape[0]:
        raise InvalidArgument("spmm: inner dimensions do not match")
    out = torch.empty((s.rows, y.shape[1]), dtype=torch.float32, device="cuda")
    check(lib().xg_spmm_f32(s.rows, s.cols, _p(s.row_ptr), _p(s.col_idx), _p(s.values), _p(y),
                            y.shape[1], _p(out), _s()))
    return out


# ---- pipeline.hpp -----------------------------------------------------------
def get_avg_vectors(d):
    x, host = _dev(d, torch.float32)
    r = torch.empty(x.shape[0], dtype=torch.float32, device="cuda")
    c = torch.empty(x.shape[1], dtype=torch.float32, device="cuda")
    check(lib().xg_avg_vectors(_p(x), x.shape[0], x.shape[1], _p(r), _p(c), _s()))
    return _ret(r, host), _ret(c, host)


def get_abs_min_vectors(d):
    x, host = _dev(d, torch.float32)
    r = torch.empty(x.shape[0], dtype=torch.float32, device="cuda")
    c = torch.empty(x.shape[1], dtype=torch.float32, device="cuda")
    check(lib().xg_abs_min_vectors(_p(x), x.shape[0], x.shape[1], _p(r), _p(c), _s()))
    return _ret(r, host), _ret(c, host)


def _fast_dev(x) -> bool:  # already a contiguous fp32 CUDA tensor: used as is
    return isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()


def _overlaps(x: torch.Tensor, y: torch.Tensor | None) -> bool:
    if y is None or x.device != y.device:
        return False
    x0, y0 = x.data_ptr(), y.data_ptr()
    return x0 < y0 + y.numel() * y.element_size() and y0 < x0 + x.numel() * x.element_size()


def _check_out(out, m: int, n: int, a: torch.Tensor, b: torch.Tensor) -> None:
    """`out` receives the result and is the pipeline's D_F scratch: a contiguous
    float32 CUDA tensor of the result's shape, not overlapping A or B."""
    if not isinstance(out, torch.Tensor) or not out.is_cuda or out.dtype != torch.float32 \
            or tuple(out.shape) != (m, n) or not out.is_contiguous():
        raise InvalidArgument("xigemm: out must be a contiguous float32 CUDA tensor of shape (M, N)")
    if _overlaps(out, a) or _overlaps(out, b):
        raise InvalidArgument("xigemm: out must not overlap A or B")


def _pipeline(a, b, c, alpha, beta, cfg: XigemmConfig, reduce: bool, dump: bool, out=None):
    if _fast_dev(a) and _fast_dev(b):
        x, host, y = a, False, b
    else:
        x, host = _dev(a, torch.float32)
        y, _ = _dev(b, torch.float32)
    if x.dim() != 2 or y.dim() != 2 or x.shape[1] != y.shape[0]:
        raise InvalidArgument("xigemm: inner dimensions do not match")
    m, k = x.shape
    n = y.shape[1]
    cc = None
    if c is not None:
        cc, _ = _dev(c, torch.float32)
        if tuple(cc.shape) != (m, n):
            raise InvalidArgument("xigemm: C shape does not match the result")
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    else:
        _check_out(out, m, n, x, y)
        if _overlaps(out, cc):  # BLAS-style in place (out is C): D_F lands in out first
            cc = cc.clone()
    rep = XgReport()
    dmp = None
    bufs = None
    if dump:
        vw = cfg.scheme == QuantScheme.VectorWise
        e = dict(device="cuda")
        bufs = dict(aq=torch.empty((m, k), dtype=torch.int8, **e),
                    aq_scales=torch.empty(m if vw else 1, dtype=torch.float64, **e),
                    bq=torch.empty((k, n), dtype=torch.int8, **e),
                    bq_scales=torch.empty(n if vw else 1, dtype=torch.float64, **e),
                    d_f=torch.empty((m, n), dtype=torch.float32, **e),
                    raq=torch.empty((m, k), dtype=torch.int8, **e),
                    raq_scale=torch.empty(1, dtype=torch.float64, **e),
                    rbq=torch.empty((k, n), dtype=torch.int8, **e),
                    rbq_scale=torch.empty(1, dtype=torch.float64, **e),
                    row_stat=torch.empty(m, dtype=torch.float32, **e),
                    col_stat=torch.empty(n, dtype=torch.float32, **e),
                    a_red=torch.empty((m, k), dtype=torch.int8, **e),
                    b_red=torch.empty((k, n), dtype=torch.int8, **e),
                    a_red_scale=torch.empty(1, dtype=torch.float64, **e),
                    b_red_scale=torch.empty(1, dtype=torch.float64, **e),
                    a_keep=torch.empty((m, (k + 31) // 32), dtype=torch.int32, **e),
                    b_keep=torch.empty((n, (k + 31) // 32), dtype=torch.int32, **e))
        dmp = XgDump(*[bufs[f].data_ptr() for f in DUMP_FIELDS])
    cfgc = cfg.c()
    check(lib().xg_xigemm(_p(x), _p(y), _p(cc), float(alpha), float(beta), m, k, n,
                          C.byref(cfgc), int(reduce), _p(out), C.byref(rep),
                          C.byref(dmp) if dmp is not None else None, _s()))
    report = GemmReport(_ret(out, host), rep.density_a, rep.density_b, GemmPath(rep.path),
                        {"quant": int(rep.ns_quant), "xxmm": int(rep.ns_xxmm),
                         "reduce": int(rep.ns_reduce), "package": int(rep.ns_package)},
                        rep.nnz_a, rep.nnz_b, rep.stats_fallbacks, rep.comp_kernel)
    report.timings["gemm_df"] = int(rep.ns_gemm_df)
    report.timings["gemm_comp"] = int(rep.ns_gemm_comp)
    return (report, bufs) if dump else report


@dataclass
class EtaCalibration:               # calibrate.hpp:15-20
    eta: float = 0.0
    repetitions: int = 1
    timer_coarse_warning: bool = False
    fingerprint: str = ""
    gemm_ops_per_s: float = 0.0     # measured tcgen05 GEMM rate (int8 op/s)
    spmm_macs_per_s: float = 0.0    # measured CSR SpMM rate near eta (MAC/s)


def calibrate_eta(size: int, bits=QuantBits.Int8, seed: int = 0, install: bool = False) -> EtaCalibration:
    """calibrate.cpp:68-100 on the device: the density where the CSR spmm_int costs as
    much as the tcgen05 gemm_int at size x size.  install=True makes the measured rates
    the SparseResidual branch's compensation cost model (comp_model)."""
    eta, reps, ptc, psp = C.c_double(), C.c_int(), C.c_double(), C.c_double()
    check(lib().xg_calibrate_eta(int(size), int(bits), int(seed) & (2 ** 64 - 1), int(bool(install)),
                                 C.byref(eta), C.byref(reps), C.byref(ptc), C.byref(psp)))
    name = torch.cuda.get_device_name() if torch.cuda.is_available() else "no-gpu"
    return EtaCalibration(eta.value, reps.value, False, name, ptc.value, psp.value)


def comp_model(p_tc: float = 0.0, p_sp: float = 0.0, bw: float = 0.0, force: int = -1) -> dict:
    """Sets (values > 0 / force >= 0) and returns the compensation cost model: the
    device chooses the tcgen05 masked-dense launch or the CUDA-core CSR SpMM for the
    sparse terms (force: 0 auto, 1 dense, 2 CSR).  Results are identical either way."""
    check(lib().xg_comp_model_set(float(p_tc), float(p_sp), float(bw), int(force)))
    v = [C.c_double(), C.c_double(), C.c_double(), C.c_int()]
    lib().xg_comp_model_get(*[C.byref(x) for x in v])
    return {"p_tc": v[0].value, "p_sp": v[1].value, "bw": v[2].value, "force": v[3].value}


def xigemm(a, b, c=None, alpha: float = 1.0, beta: float = 0.0, cfg: XigemmConfig | None = None,
           *, out=None) -> GemmReport:
    """pipeline.hpp:57-62: D = alpha*A*B(compensated) + beta*C."""
    return _pipeline(a, b, c, alpha, beta, cfg or XigemmConfig(), True, False, out)


def xigemm_dump(a, b, cfg: XigemmConfig | None = None):
    """xigemm plus every intermediate in the reference's layouts (parity tests)."""
    return _pipeline(a, b, None, 1.0, 0.0, cfg or XigemmConfig(), True, True)


def quantized_gemm_full_residual(a, b, cfg: XigemmConfig | None = None, *, out=None):
    """pipeline.hpp:50-51 / pipeline.cpp:177-180 (out=: as for xigemm)."""
    return _pipeline(a, b, None, 1.0, 0.0, cfg or XigemmConfig(), False, False, out=out).result


def quantized_gemm_direct(a, b, cfg: XigemmConfig | None = None):
    cfg = cfg or XigemmConfig()
    if isinstance(a, QuantizedMatrix):
        aq, bq = a, b
        if aq.cols != bq.rows:
            raise InvalidArgument("gemm_int: inner dimensions do not match")
        out = torch.empty((aq.rows, bq.cols), dtype=torch.float32, device="cuda")
        check(lib().xg_gemm_direct_q(_p(aq.data), int(aq.scales.scheme), _p(_scales_dev(aq.scales)),
                                     _p(bq.data), int(bq.scales.scheme), _p(_scales_dev(bq.scales)),
                                     aq.rows, aq.cols, bq.cols, int(aq.bits), int(bq.bits),
                                     _p(out), _s()))
        return out
    x, host = _dev(a, torch.float32)
    y, _ = _dev(b, torch.float32)
    if x.shape[1] != y.shape[0]:
        raise InvalidArgument("quantized_gemm_direct: inner dimensions do not match")
    out = torch.empty((x.shape[0], y.shape[1]), dtype=torch.float32, device="cuda")
    cfgc = cfg.c()
    check(lib().xg_gemm_direct(_p(x), _p(y), x.shape[0], x.shape[1], y.shape[1], C.byref(cfgc),
                               _p(out), _s()))
    return _ret(out, host)


def xigemm_host(a: np.ndarray, b: np.ndarray, c=None, alpha=1.0, beta=0.0,
                cfg: XigemmConfig | None = None, reduce=True, out=None):
    """Host-buffer entry point (xg_xigemm_host): H2D, pipeline, D2H in one call."""
    cfg = cfg or XigemmConfig()
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise InvalidArgument("xigemm: inner dimensions do not match")
    m, k = a.shape
    n = b.shape[1]
    if out is None:
        out = np.empty((m, n), np.float32)
    elif not isinstance(out, np.ndarray) or out.dtype != np.float32 or out.shape != (m, n) \
            or not out.flags.c_contiguous or not out.flags.writeable:
        raise InvalidArgument("xigemm: out must be a writable C-contiguous float32 array of shape (M, N)")
    if np.shares_memory(out, a) or np.shares_memory(out, b):
        raise InvalidArgument("xigemm: out must not overlap A or B")
    cp = None
    if c is not None:
        c = np.ascontiguousarray(c, np.float32)
        if c.shape != (m, n):  # pipeline.cpp:185-187
            raise InvalidArgument("xigemm: C shape does not match the result")
        if np.shares_memory(c, out):
            c = c.copy()
        cp = c.ctypes.data
    rep = XgReport()
    cfgc = cfg.c()
    check(lib().xg_xigemm_host(C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data),
                               C.c_void_p(cp), float(alpha), float(beta), m, k, n, C.byref(cfgc),
                               int(reduce), C.c_void_p(out.ctypes.data), C.byref(rep)))
    return out, rep


# ---- synthetic inputs -------------------------------------------------------------
def generate(kind: str, rows: int, cols: int, seed: int, p1: float = 0.0, p2: float = 1.0,
             out: torch.Tensor | None = None) -> torch.Tensor:
    """Device-side SplitMix64 generator: kind 'uniform' (lo=p1, hi=p2; bit-identical
    to test_support.hpp:16-24), 'normal' (mean p1, std p2), 'student_t3' (scale p2),
    'exponential' (rate p1)."""
    kinds = {"uniform": 0, "normal": 1, "student_t3": 2, "exponential": 3}
    if out is None:
        out = torch.empty((rows, cols), dtype=torch.float32, device="cuda")
    check(lib().xg_generate(kinds[kind], float(p1), float(p2), seed, rows * cols, _p(out), _s()))
    return out
