// Shared device helpers for the sm_100a kernels of the compensated INT8 GEMM.
//
//  * exact scalar rules of the reference (Appendix A of SURVEY.md): every fp64 /
//    fp32 operation that the reference performs is issued with an explicit
//    round-to-nearest intrinsic so nvcc can never contract it into an FMA;
//  * thin inline-PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor), and the
//    5th-generation tensor core (tcgen05.* with TMEM accumulators).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace xg {

// Enum encodings follow the reference declaration order.
enum Rounding : int { kFloor = 0, kNearest = 1 };                       // quantize.hpp:18
enum Scheme : int { kPerTensor = 0, kPerRow = 1, kPerColumn = 2 };      // quantize.hpp:20
enum QScheme : int { kQTensor = 0, kQVector = 1 };                      // pipeline.hpp:15
enum Policy : int { kAvg = 0, kMin = 1 };                               // sparse.hpp:40
enum Path : int { kSparse = 0, kDense = 1 };                            // pipeline.hpp:30

constexpr int kNumSMs = 148;

__host__ __device__ inline int quant_max(int bits) { return (1 << (bits - 1)) - 1; }
__host__ __device__ inline int gemm_max_inner(int bits) { return 1 << (31 - 2 * bits - 1); }

// quantize.cpp:99-105 — caller guarantees max_abs finite and >= 0.
__device__ __forceinline__ double compute_scale(double max_abs, int bits) {
    return max_abs == 0.0 ? 1.0 : __ddiv_rn((double)quant_max(bits), max_abs);
}

// quantize.cpp:13-24.  llround (ties away from zero) or the "Floor" path
// (4-eps nudge away from zero, then truncation).  Out-of-range conversions
// reproduce x86-64's LLONG_MIN result, which the clamp sends to -qmax.
__device__ __forceinline__ int quantize_scalar(double a, double lambda, int qmax, int rounding) {
    double t = __dmul_rn(a, lambda);
    if (rounding == kFloor) {
        const double nudge = __dmul_rn(4.0 * 2.220446049250313080847e-16, fabs(t));
        t = __dadd_rn(t, copysign(nudge, t));
        if (!(fabs(t) < 9223372036854775808.0)) return -qmax;
        t = trunc(t);
    } else {
        if (!(fabs(t) < 9223372036854775808.0)) return -qmax;
        t = round(t);  // half away from zero == llround
    }
    if (t < -(double)qmax) return -qmax;
    if (t > (double)qmax) return qmax;
    return (int)t;
}

// Pipeline-only fast form of quantize_scalar, valid when |a*lambda| < 2^63
// (always true inside the pipeline: lambda = qmax / max|slice| and |a| <= max,
// so |t| <= qmax (1 + 2^-52)).  Clamping before rounding is then identical to
// the reference's round-then-clamp, NaN clamps to -qmax like x86's LLONG_MIN,
// and llround's ties-away is restored from rint's ties-even with an exact
// correction.  ~8 instructions instead of libdevice round() + range tests.
__device__ __forceinline__ int quantize_fast(double a, double lambda, double qmax_d, int rounding) {
    double t = __dmul_rn(a, lambda);
    if (rounding == kFloor) {
        t = __dadd_rn(t, copysign(__dmul_rn(4.0 * 2.220446049250313080847e-16, fabs(t)), t));
        t = fmin(fmax(t, -qmax_d), qmax_d);
        return (int)t;  // truncation toward zero
    }
    t = fmin(fmax(t, -qmax_d), qmax_d);
    double r = rint(t);
    if (fabs(__dsub_rn(t, r)) == 0.5) r = __dadd_rn(t, copysign(0.5, t));
    return (int)r;
}

// fp32 fast path with an exact fallback.  With lam32 = RN_f(lambda),
// t32 = RN_f(a * lam32) differs from the reference's t = RN_d(a * lambda) by at
// most |t| * 2^-23 (+ 2^-53) <= 1.6e-5 for |t| <= 128.  Nearest: llround(t)
// equals rint(t32) unless t32 lies within 1e-4 of a half-integer; Floor:
// trunc(t + nudge) equals trunc(t32) unless t32 lies within 2e-4 of an integer.
// Those rare cases (~2e-4 of elements) take the exact fp64 path.  The rounding
// itself uses the 1.5*2^23 magic constant, whose float bits hold the integer in
// the low byte (two's complement), so no float->int conversion is needed.
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
// out-of-line so the rare exact path does not bloat every inlined call site
static __device__ __noinline__ int quantize_slow(float a, double lambda, float qmaxf, int rounding) {
    return quantize_fast((double)a, lambda, (double)qmaxf, rounding);
}
__device__ __forceinline__ int quantize32(float a, double lambda, float lam32, float qmaxf,
                                          int rounding) {
    const float t0 = __fmul_rn(a, lam32);
    const float t = fminf(fmaxf(t0, -qmaxf), qmaxf);
    const bool wild = !(fabsf(t0) <= 256.0f);  // NaN input, or lambda outside float range
    if (rounding == kFloor) {
        const float r = truncf(t);
        const float d = fabsf(__fsub_rn(t, r));
        if (wild || d < 2e-4f || d > 0.9998f) return quantize_slow(a, lambda, qmaxf, rounding);
        return (int)r;
    }
    const float u = __fadd_rn(t, kMagic);
    const float r = __fsub_rn(u, kMagic);
    if (wild || fabsf(__fsub_rn(t, r)) >= 0.4999f) return quantize_slow(a, lambda, qmaxf, rounding);
    return __float_as_int(u) - 0x4B400000;
}

// Smallest float strictly greater than the fp64 threshold t >= 0, so that the
// reference's keep test fabs(double(v)) > t (sparse.cpp:65) becomes the float
// compare |v| >= float_above(t) for float v.
__device__ __forceinline__ float float_above(double t) {
    float f = __double2float_ru(t);
    if ((double)f == t) f = nextafterf(f, __int_as_float(0x7f800000));
    return f;
}

// float(double(q) / lambda) — quantize.cpp:156.
__device__ __forceinline__ float dequant_value(int q, double lambda) {
    return __double2float_rn(__ddiv_rn((double)q, lambda));
}

// float(double(p) / (la * lb)) — quantize.cpp:183.
__device__ __forceinline__ float dequant_product_value(int32_t p, double la, double lb) {
    return __double2float_rn(__ddiv_rn((double)p, __dmul_rn(la, lb)));
}

// ---- fast exact dequantisation -------------------------------------------
// The reference rounds twice: q = RN_d(p / RN_d(la*lb)), then RN_f(q).  We
// form y = RN(RN(p * ia) * ib) with ia = RN(1/la), ib = RN(1/lb); |y - q| is a
// few double ulps (<= ~6u|y|).  RN_f is monotone, so when y lies more than 64
// double ulps away from every float rounding boundary (a float midpoint sits
// where the 29 discarded mantissa bits equal 2^28) and inside the float normal
// range, RN_f(y) == RN_f(q) exactly.  Otherwise (probability ~2e-7) fall back
// to the reference's own division.  Zero products are exact (+0).
__device__ __forceinline__ bool float_round_safe(double y) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(y);
    const unsigned e = (unsigned)(b >> 52) & 0x7ffu;
    const int low = (int)((unsigned)b & 0x1fffffffu) - 0x10000000;
    return e >= 1023u - 126u && e <= 1023u + 126u && (low > 64 || low < -64);
}
__device__ __forceinline__ float dequant_product_fast(int32_t p, double ia, double ib, double la,
                                                      double lb) {
    if (p == 0) return 0.0f;
    const double y = __dmul_rn(__dmul_rn((double)p, ia), ib);
    if (float_round_safe(y)) return __double2float_rn(y);
    return dequant_product_value(p, la, lb);
}
// Same with the column scale fetched only on the (rare) slow path.
__device__ __forceinline__ float dequant_product_fast2(int32_t p, double ia, double ib, double la,
                                                       const double* lb_ptr) {
    if (p == 0) return 0.0f;
    const double y = __dmul_rn(__dmul_rn((double)p, ia), ib);
    if (float_round_safe(y)) return __double2float_rn(y);
    return dequant_product_value(p, la, *lb_ptr);
}
// Conversion-free variant.  On this part I2F.F64 and F2F.F32.F64 issue at
// ~16 and ~12 per clock per SM (measured, tools/microbench/pipes.cu) against
// 62 DMUL, so: p -> double exactly via the 2^52 + 2^31 magic constant (one
// DADD), and once float_round_safe has proven y is not near a float rounding
// boundary, RN_f(y) is assembled from y's bits with integer ops (exponent
// rebias by xor, 23-bit mantissa by a funnel shift, round bit added with carry).
// Returns the float; sets `slow` if the exact division is required.
__device__ __forceinline__ float dq_bits(int32_t p, double ia, double ib, bool& slow) {
    const double pd = __dsub_rn(__hiloint2double(0x43300000, (int)((uint32_t)p ^ 0x80000000u)),
                                4503601774854144.0);  // 2^52 + 2^31
    const double y = __dmul_rn(__dmul_rn(pd, ia), ib);
    const uint32_t hi = (uint32_t)__double2hiint(y), lo = (uint32_t)__double2loint(y);
    const uint32_t e = (hi >> 20) & 0x7ffu;
    const int low = (int)(lo & 0x1fffffffu) - 0x10000000;
    const bool ok = e >= 1023u - 126u && e <= 1023u + 126u && (low > 64 || low < -64);
    slow |= !ok && p != 0;
    uint32_t f = __funnelshift_l(lo, hi, 3);                     // hi[28:0] . lo[31:29]
    f = ((f ^ 0x40000000u) & 0x7fffffffu) | (hi & 0x80000000u);  // exponent 1023 -> 127 bias
    f += (lo >> 28) & 1u;                                        // round to nearest (not a tie)
    return p == 0 ? 0.0f : __uint_as_float(f);
}

// FP64-free variant for the tensor-core epilogues.  On B200 DMUL/DADD issued
// by the epilogue warps slow the concurrently running tcgen05.mma by ~20%
// (tools/gemm_ceiling.py: 426 us with dq_bits vs 352 us without dequant math,
// 354 us with fp32 math of the same shape), so the exact dequantisation runs in
// float-float arithmetic:
//   1/la ~ ah + al, 1/lb ~ bh + bl            (ff_recip, once per row/column)
//   c = (ah+al)(bh+bl) ~ ch + cl              (|rel err| < 2^-45)
//   p = ph + pl, ph = p & ~255, pl = p & 255  (both exact floats)
//   y = p*c = s + lo with ph*ch, pl*ch exact (FMA) and Fast2Sum
//   f = RN_f(s + lo); r = (s - f) + lo  (signed distance y - f, Sterbenz-exact)
// The reference's q = RN_d(p / RN_d(la*lb)) is within 2^-51|q| of p/(la*lb);
// y is within 2^-42.5|y|.  If |r| + 2^(E-40) < 2^(E-24) (half an ulp of f,
// E = f's biased exponent) both lie strictly on f's side of the float
// midpoints, so RN_f(q) == f.  Powers of two (the ulp halves below them),
// tiny/huge values and non-finite scales fall back to the exact division
// (probability ~2^-16 per element).  Zero products give +0 like the reference.
__device__ __forceinline__ float2 ff_recip(double lam) {
    const double ia = __ddiv_rn(1.0, lam);
    const float h = __double2float_rn(ia);
    const float l = __double2float_rn(__dsub_rn(ia, (double)h));
    const float ah = fabsf(h);
    // keep ch = ah*bh in [2^-100, 2^100] so cl and the FMA error terms stay normal
    if (!(ah >= 0x1p-50f && ah <= 0x1p50f)) return make_float2(__int_as_float(0x7fc00000), 0.0f);
    return make_float2(h, l);
}

__device__ __forceinline__ float dq_ff(int32_t p, float2 a, float2 b, bool& slow) {
    // the reference's 0 / (la*lb) with la*lb positive and finite (compute_scale's
    // range), also when a scale is outside ff_recip's range (NaN marker)
    if (p == 0) return 0.0f;
    const float ch = __fmul_rn(a.x, b.x);
    const float ce = __fmaf_rn(a.x, b.x, -ch);
    const float cl = __fmaf_rn(a.x, b.y, __fmaf_rn(a.y, b.x, ce));
    const int32_t phi = p & ~255;
    const float ph = __int2float_rn(phi);                                          // exact: 23 bits
    const float pl = __fsub_rn(__int_as_float(0x4b000000 | (p & 255)), 8388608.0f);  // exact: 8 bits
    const float t1 = __fmul_rn(ph, ch);
    const float e1 = __fmaf_rn(ph, ch, -t1);
    const float t3 = __fmul_rn(pl, ch);
    const float e3 = __fmaf_rn(pl, ch, -t3);
    const float s = __fadd_rn(t1, t3);  // Fast2Sum: |t1| >= |t3| or t1 == 0
    const float es = __fsub_rn(t3, __fsub_rn(s, t1));
    const float lo = __fadd_rn(__fmaf_rn(ph, cl, __fmaf_rn(pl, cl, e3)), __fadd_rn(e1, es));
    const float f = __fadd_rn(s, lo);
    const float r = __fadd_rn(__fsub_rn(s, f), lo);
    const uint32_t fb = __float_as_uint(f);
    const uint32_t ef = fb & 0x7f800000u;
    const float half = __uint_as_float(ef - (24u << 23));
    const float marg = __uint_as_float(ef - (40u << 23));
    const bool ok = ef >= (42u << 23) && ef <= (253u << 23) && (fb & 0x007fffffu) != 0u &&
                    __fadd_rn(fabsf(r), marg) < half;
    slow |= !ok && p != 0;
    return f;
}

// Epilogue fast form for |p| < 2^24 (p exact as a float, the common case: a
// K=8192 int8 product of random data stays near 1e5): y = pf*(ch + cl) with
// pf*ch exact as t1 + e1, |y - p/(la*lb)| <= 2^-44.5|y|.  Accepted when
// |r| <= 2^(e-24) - 2^(e-39), e the exponent of the float just below |f|:
// half the gap to f's lower neighbour minus a margin 8x the error bound, so y
// and the reference's q lie strictly on f's side of both neighbouring
// midpoints (for a power of two f the lower gap is ulp(f)/2, and e is one
// less).  No range tests are needed: ff_recip's ranges give ch in
// [2^-100, 2^100], so for 0 < |p| < 2^24 f is normal and finite and every
// error term is exact or far below the margin; p = 0 gives f = r = +0
// (accepted: the reference's +0); a non-finite scale marker makes r NaN
// (rejected).  Elements that fail (|p| >= 2^24, ~2^-15 of random ones) set
// their bit in `slowmask` and are redone by dq_slow.
// c = (ah + al)(bh + bl) as ch + cl (the scale product of dq_ff24, hoistable
// when one scale is fixed over many elements)
__device__ __forceinline__ float2 ff_mul(float2 a, float2 b) {
    const float ch = __fmul_rn(a.x, b.x);
    const float ce = __fmaf_rn(a.x, b.x, -ch);
    return make_float2(ch, __fmaf_rn(a.x, b.y, __fmaf_rn(a.y, b.x, ce)));
}

__device__ __forceinline__ float dq_ff24c(int32_t p, float2 c, uint32_t& slowmask, uint32_t bit) {
    const float ch = c.x, cl = c.y;
    const float pf = __int2float_rn(p);
    const float t1 = __fmul_rn(pf, ch);
    const float e1 = __fmaf_rn(pf, ch, -t1);
    const float lo = __fmaf_rn(pf, cl, e1);
    const float f = __fadd_rn(t1, lo);
    const float r = __fadd_rn(__fsub_rn(t1, f), lo);
    // exponent of the float just below |f| (fb - 1): one less than f's own for a
    // power of two, whose lower neighbour is only ulp(f)/2 away
    const int ef = (int)((__float_as_uint(f) - 1u) & 0x7f800000u);
    const float thr = __int_as_float(max(ef - ((24 << 23) + 256), 0));
    const bool ok = fabsf(pf) < 16777216.0f && fabsf(r) <= thr;
    slowmask |= ok ? 0u : bit;
    return f;
}

// Packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2 on sm_100a): two IEEE
// round-to-nearest operations per instruction, each lane's result identical to
// the scalar operation's (tools/microbench/f32x2_check.cu).  Caution: ptxas
// contracts a packed mul feeding a packed add/sub into one FFMA2 even with .rn
// (tools/microbench/dq2_check.cu), so a product must only ever reach an FMA as
// its addend; the users here (quant.cu qn4) have no such pair.
__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__device__ __forceinline__ float dq_ff24(int32_t p, float2 a, float2 b, uint32_t& slowmask,
                                         uint32_t bit) {
    return dq_ff24c(p, ff_mul(a, b), slowmask, bit);
}

// Rare path of the epilogues: the full-range float-float form, then the
// reference's own fp64 division.
static __device__ __noinline__ float dq_slow(int32_t p, float2 a, float2 b, double la, double lb) {
    bool slow = false;
    const float f = dq_ff(p, a, b, slow);
    return slow ? dequant_product_value(p, la, lb) : f;
}

// float(q / lambda) with il = RN(1/lambda)
__device__ __forceinline__ float dequant_fast(int q, double il, double lambda) {
    if (q == 0) return 0.0f;
    const double y = __dmul_rn((double)q, il);
    if (float_round_safe(y)) return __double2float_rn(y);
    return dequant_value(q, lambda);
}

// Non-negative float <-> order-preserving uint bits (for atomicMax / atomicMin).
__device__ __forceinline__ uint32_t fbits(float x) { return __float_as_uint(x); }

// ---------------------------------------------------------------- warp ops --
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_maxf(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sumd(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Programmatic dependent launch: a kernel that may be started before its
// predecessor in the graph has finished (programmatic edge) waits here before
// touching any memory the predecessor writes.  A no-op without such an edge.
// Programmatic dependent launch: wait for the predecessor grid (and its
// memory), then let the successor grid launch at once - its CTAs run their
// prologue where resources free up and park in their own wait, instead of
// being launched only when this grid has exited.  XG_PDL_EARLY=0 at build
// time keeps the implicit trigger at grid completion.
#ifndef XG_PDL_EARLY
#define XG_PDL_EARLY 1
#endif
#if XG_PDL_EARLY
#define XG_PDL_WAIT() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")
#else
#define XG_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#endif
// wait only (successor launched at grid completion): the persistent GEMMs
#define XG_PDL_WAIT_ONLY() asm volatile("griddepcontrol.wait;" ::: "memory")

// --------------------------------------------------------------- PTX: misc --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// ------------------------------------------------------------ PTX: mbarrier --
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t a, uint32_t parity) {
    uint32_t ok = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Blocking wait with a hang guard: a pipeline bug turns into a trapped launch
// (cudaErrorLaunchFailure) after 20 s instead of a wedged GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    if (mbar_try_wait(a, parity)) return;
    const uint64_t t0 = global_ns();
    while (!mbar_try_wait(a, parity)) {
        if (global_ns() - t0 > 20000000000ull) __trap();
    }
}

// ----------------------------------------------------------------- PTX: TMA --
__device__ __forceinline__ void tma_prefetch(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int x,
                                            int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// 1-D bulk copy global -> shared (size and addresses multiples of 16 bytes).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// order prior generic-proxy shared accesses before subsequent async-proxy ones
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMA 2-D store shared -> global (bulk-group completion).
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tmap),
                 "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N committed bulk groups still read their shared source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------------ PTX: tcgen05 --
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Arrive on `bar` once every previously issued tcgen05.mma of this thread retires.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
// D[tmem] (+)= A[smem] x B[smem]^T, int8 x int8 -> s32, one CTA.
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// ---- CTA-pair (cta_group::2) variants ------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// max into a u32 in another CTA's shared memory (shared::cluster address)
__device__ __forceinline__ void red_max_cluster_u32(uint32_t cluster_addr, uint32_t v) {
    asm volatile("red.relaxed.cluster.shared::cluster.max.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_cluster_u32(uint32_t cluster_addr) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(cluster_addr) : "memory");
    return v;
}
// shared::cluster address of `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
// Arrive on a barrier of another CTA of the cluster (the pair leader's TMEM
// "empty" barriers).  Default .release.cta semantics: what it publishes is
// TMEM reads, ordered by tcgen05.fence::before_thread_sync, not generic
// memory, so no cluster-scope release fence (MEMBAR.ALL.GPU) is needed.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
                 : "memory");
}
// TMA load whose completion is counted on the LEADER CTA's barrier (peer bit
// of the shared::cta barrier address cleared).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, uint64_t* bar, int x,
                                                 int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y)
        : "memory");
}
// L2-only prefetch of a 2-D tensor box (no shared memory, no barrier): hides
// DRAM latency for loads issued later from the same box.
__device__ __forceinline__ void tma_prefetch_l2(const void* tmap, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tmap), "r"(x),
                 "r"(y)
                 : "memory");
}
// 2SM TMA load multicast to the CTAs in `mask`; completion is counted on the
// pair-leader barrier of each destination.
__device__ __forceinline__ void tma_load_2d_pair_mc(void* dst, const void* tmap, uint64_t* bar, int x, int y,
                                                    uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y), "h"(mask)
        : "memory");
}
// commit arriving on the barrier at the same offset in every CTA of `mask`
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// commit arriving on the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets lane
// (warp%4)*32+t, columns [col, col+32).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}
template <int W>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[W]) {
    if constexpr (W == 32) tmem_ld32(taddr, r);
    else tmem_ld16(taddr, r);
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor for a K-major operand tile written by TMA
// with 128-byte swizzling: rows of 128 bytes, 8-row (1024 B) swizzle atoms.
//   bits  0-13 start address >> 4
//   bits 16-29 leading byte offset >> 4 (unused for swizzled K-major; 1)
//   bits 32-45 stride byte offset >> 4 (1024 B between 8-row groups)
//   bits 46-47 descriptor version (1 on sm_100)
//   bits 61-63 layout: 2 = SWIZZLE_128B
__device__ __forceinline__ uint64_t smem_desc_k128(const void* p) {
    const uint64_t addr = smem_u32(p);
    return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) | ((1024ull >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}

// Instruction descriptor: s32 accumulator, signed int8 A and B, both K-major.
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
    return (2u << 4)             // D format s32
           | (1u << 7)           // A signed 8-bit
           | (1u << 10)          // B signed 8-bit
           | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

}  // namespace xg
