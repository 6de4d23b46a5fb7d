// Sparse compensation path: the reference's CSR formulation of dr1 = A'q RBq
// and dr2 = RAq B'q (sparse.cpp:119-138, pipeline.cpp:118-124) on CUDA cores,
// for residual densities where it beats the masked-dense tensor-core launch
// (the device-side choice in k_dispatch, calibrated by xg_calibrate_comp).
//
//   k_qcsr_build   masked int8 operand (A'q rows / B'q^T rows, K-major) ->
//                  quad-packed CSR: per row a (first quad, quads) segment of
//                  4-entry groups {4 x uint16 k, 4 x int8 v}, zero-padded.
//                  Stream compaction, one warp per row: per-lane non-zero
//                  counts, a warp scan (shuffles) for the offsets, one atomic
//                  per 8-row block for the block's segments.
//   k_spmm_strip   persistent CUDA-core SpMM: a CTA stages a strip of W dense
//                  lines x K (W x K int8, K-major lines: RBq^T rows for dr1,
//                  RAq rows for dr2) transposed into shared memory as
//                  strip[k][W] (128 KiB), then every lane walks one sparse
//                  row's quads: 4 strip rows (LDS.128 / LDS.64), a 4x4 byte
//                  transpose (PRMT) and IDP4A per 4 columns - 4 exact int8
//                  MACs per instruction.  The staged strip is reused by all
//                  sparse rows of the CTA's items (strip-major work order).
//                  Epilogues: raw s32 (spmm_int), out = fl(din + deq(acc))
//                  (dr1, pipeline.cpp:141-143) and the transposed
//                  out = fl(out + deq(acc)) + alpha/beta (dr2,
//                  pipeline.cpp:144-145, :195-202) with the GEMM epilogue's
//                  exact dequantisation (common.cuh dq_ff24 / dq_slow).
//
// Integer sums are exact and order-free, so the result is bit-identical to the
// masked-dense path and to the reference; entries whose quantised value is 0
// are not stored (they add 0).
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "spmm.h"

namespace xg {
namespace {

constexpr int kBuildWarps = 8;
constexpr int kBuildRows = 8;  // k_qcsr_from_csr: rows per warp per block (64 rows per CTA)

// entry p of the quad array (entry p % 4 of quad p / 4)
__device__ __forceinline__ void put_entry(uint4* quad, int64_t p, int k, int8_t v) {
    uint8_t* rec = reinterpret_cast<uint8_t*>(quad + (p >> 2));
    reinterpret_cast<uint16_t*>(rec)[p & 3] = (uint16_t)k;
    reinterpret_cast<int8_t*>(rec + 8)[p & 3] = v;
}

// bit 8b+7 set iff byte b of w is non-zero (3 integer ops)
__device__ __forceinline__ uint32_t nz_mask(uint32_t w) { return (((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) & 0x80808080u; }
__device__ __forceinline__ int nz_bytes(uint32_t w) { return __popc(nz_mask(w)); }

__device__ __forceinline__ uint4 ld_row16(const int8_t* p, int valid) {
    uint4 v = *reinterpret_cast<const uint4*>(p);
    if (valid < 16) {  // bytes past the row's end (pitch padding) are not data
        uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int keep = min(max(valid - 4 * i, 0), 4);
            w[i] &= keep >= 4 ? 0xffffffffu : ((1u << (8 * keep)) - 1u);
        }
    }
    return v;
}

// x: rows x cols int8, row pitch ld (multiple of 16).  One warp per row: the
// row's non-zeros are counted (8 x 16 bytes per lane in flight), the row's
// segment is reserved with one atomic, then the row is re-read (L1/L2) and
// compacted in ascending k: per 512-column chunk each lane's count, a warp
// inclusive scan (shuffles) for its offsets, the non-zero bytes scattered.
// run: device flag, the kernel returns at once when *run == 0 (the dense launch
// serves the call); bad: raised when the buffer (or max_quads) is exceeded.
constexpr int kBatch = 8;  // 512-column chunks per batch of loads

__global__ void __launch_bounds__(kBuildWarps * 32)
    k_qcsr_build(const int8_t* __restrict__ x, int rows, int cols, int64_t ld, QCsr q, const int* run,
                 int* bad, int max_quads) {
    XG_PDL_WAIT();
    if (run && !*run) return;
    __shared__ int cnt[kBuildWarps];
    __shared__ long long first[kBuildWarps];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int rb = blockIdx.x * kBuildWarps; rb < rows; rb += gridDim.x * kBuildWarps) {
        const int r = rb + w;
        const int8_t* row = x + (int64_t)r * ld;
        int c = 0;
        if (r < rows) {
            for (int cb = 0; cb < cols; cb += 512 * kBatch) {
                uint4 v[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int c0 = cb + u * 512 + lane * 16;
                    v[u] = c0 < cols ? ld_row16(row + c0, cols - c0) : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u)
                    c += nz_bytes(v[u].x) + nz_bytes(v[u].y) + nz_bytes(v[u].z) + nz_bytes(v[u].w);
            }
            c = warp_sum(c);
        }
        if (lane == 0) cnt[w] = (c + 3) >> 2;
        __syncthreads();
        if (threadIdx.x == 0) {  // the block's segments: exclusive scan + one atomic
            long long tot = 0;
            int mx = 0;
            for (int i = 0; i < kBuildWarps; ++i) {
                first[i] = tot;
                tot += cnt[i];
                mx = max(mx, cnt[i]);
            }
            const long long base = tot ? (long long)atomicAdd(q.cursor, (unsigned long long)tot) : 0ll;
            const bool over = base + tot > q.cap_q || mx > max_quads;
            if (over) atomicOr(bad, 1);
            for (int i = 0; i < kBuildWarps; ++i) first[i] = over ? -1 : first[i] + base;
        }
        __syncthreads();
        const long long q0 = first[w];
        const int nq = cnt[w];
        __syncthreads();  // cnt / first are rewritten by the next block
        if (r >= rows || q0 < 0) continue;
        if (lane == 0) q.seg[r] = make_int2((int)q0, nq);
        int64_t off = q0 * 4;
        for (int cb = 0; cb < cols; cb += 512 * kBatch) {
            uint4 v[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int c0 = cb + u * 512 + lane * 16;
                v[u] = c0 < cols ? ld_row16(row + c0, cols - c0) : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int c0 = cb + u * 512 + lane * 16;
                const int n = nz_bytes(v[u].x) + nz_bytes(v[u].y) + nz_bytes(v[u].z) + nz_bytes(v[u].w);
                if (__ballot_sync(0xffffffffu, n != 0) == 0u) continue;  // (warp-uniform) empty 512 columns
                int incl = n;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += t;
                }
                int64_t p = off + incl - n;
                const uint32_t ws[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    uint32_t m = nz_mask(ws[i]);
                    while (m) {
                        const int bb = (__ffs(m) - 1) >> 3;
                        put_entry(q.quad, p, c0 + 4 * i + bb, (int8_t)(ws[i] >> (8 * bb)));
                        ++p;
                        m &= m - 1u;
                    }
                }
                off += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        // zero padding of the last quad (k = 0 is a valid strip row)
        const int64_t end = (q0 + nq) * 4;
        if (off + lane < end) {
            put_entry(q.quad, off + lane, 0, 0);
        }
    }
}

// Standard CSR (row_ptr, int32 col_idx, int8 values) -> quad-packed rows (spmm_int API).
__global__ void __launch_bounds__(kBuildWarps * 32)
    k_qcsr_from_csr(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, const int8_t* __restrict__ v,
                    int rows, QCsr q) {
    XG_PDL_WAIT();
    __shared__ int cnt[kBuildWarps * kBuildRows];
    __shared__ int first[kBuildWarps * kBuildRows];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kBlock = kBuildWarps * kBuildRows;
    for (int rb = blockIdx.x * kBlock; rb < rows; rb += gridDim.x * kBlock) {
        if (threadIdx.x < kBlock) {
            const int r = rb + threadIdx.x;
            cnt[threadIdx.x] = r < rows ? (rp[r + 1] - rp[r] + 3) >> 2 : 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int i = 0; i < kBlock; ++i) {
                first[i] = tot;
                tot += cnt[i];
            }
            const unsigned long long base = tot ? atomicAdd(q.cursor, (unsigned long long)tot) : 0ull;
            for (int i = 0; i < kBlock; ++i) first[i] += (int)base;
        }
        __syncthreads();
        for (int j = 0; j < kBuildRows; ++j) {
            const int qi = w * kBuildRows + j, r = rb + qi;
            if (r >= rows) break;
            const int q0 = first[qi], nq = cnt[qi];
            if (lane == 0) q.seg[r] = make_int2(q0, nq);
            const int p0 = rp[r], n = rp[r + 1] - p0;
            for (int e = lane; e < nq * 4; e += 32) {
                const bool in = e < n;
                put_entry(q.quad, (int64_t)q0 * 4 + e, in ? ci[p0 + e] : 0, in ? v[p0 + e] : (int8_t)0);
            }
        }
        __syncthreads();
    }
}

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

// acc[c] += sum_t byte_c(r_t) * byte_t(v): 4 columns of one 32-bit strip word
// from 4 strip rows (the quad's k), via a 4x4 byte transpose.
__device__ __forceinline__ void mac4(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3, int v, int* acc) {
    const uint32_t t0 = __byte_perm(r0, r1, 0x5140), t1 = __byte_perm(r0, r1, 0x7362);
    const uint32_t t2 = __byte_perm(r2, r3, 0x5140), t3 = __byte_perm(r2, r3, 0x7362);
    acc[0] = __dp4a((int)__byte_perm(t0, t2, 0x5410), v, acc[0]);
    acc[1] = __dp4a((int)__byte_perm(t0, t2, 0x7632), v, acc[1]);
    acc[2] = __dp4a((int)__byte_perm(t1, t3, 0x5410), v, acc[2]);
    acc[3] = __dp4a((int)__byte_perm(t1, t3, 0x7632), v, acc[3]);
}

__device__ __forceinline__ float2 srcp(const SpScale& s, int i) {
    return s.r ? s.r[(int64_t)i * s.stride] : ff_recip(s.p[(int64_t)i * s.stride]);
}

constexpr int kHeavyQ = 64;  // quads; longer rows are shared by the warp
constexpr int kTileP = 20;   // floats per row of the epilogue staging tile (80 bytes)

// acc[0..W) += the quad's 4 entries times their W-wide strip rows
template <int W>
__device__ __forceinline__ void quad_mac(const uint4 rec, uint32_t sbase, int* acc) {
    const int vv = (int)rec.z;
    const uint32_t ad0 = sbase + (rec.x & 0xffffu) * W, ad1 = sbase + (rec.x >> 16) * W;
    const uint32_t ad2 = sbase + (rec.y & 0xffffu) * W, ad3 = sbase + (rec.y >> 16) * W;
    if constexpr (W == 16) {
        const uint4 r0 = lds128(ad0), r1 = lds128(ad1), r2 = lds128(ad2), r3 = lds128(ad3);
        mac4(r0.x, r1.x, r2.x, r3.x, vv, acc);
        mac4(r0.y, r1.y, r2.y, r3.y, vv, acc + 4);
        mac4(r0.z, r1.z, r2.z, r3.z, vv, acc + 8);
        mac4(r0.w, r1.w, r2.w, r3.w, vv, acc + 12);
    } else {
        const uint2 r0 = lds64(ad0), r1 = lds64(ad1), r2 = lds64(ad2), r3 = lds64(ad3);
        mac4(r0.x, r1.x, r2.x, r3.x, vv, acc);
        mac4(r0.y, r1.y, r2.y, r3.y, vv, acc + 4);
    }
}

// quads [q0, q0 + n) with the next record's load in flight during each MAC
// step; `first` is the record of quad q0, already loaded by the caller
template <int W>
__device__ __forceinline__ void quads_mac(const uint4* __restrict__ quad, uint4 first, int q0, int n, int step,
                                          uint32_t sbase, int* acc) {
    uint4 rec = first;
    for (int i = 0; i < n; i += step) {
        const uint4 nxt = i + step < n ? __ldg(quad + q0 + i + step) : rec;
        quad_mac<W>(rec, sbase, acc);
        rec = nxt;
    }
}

// the W x K strip of dense lines [l0, l0 + W) into shared memory as strip[k][W]
template <int W, int NT>
__device__ __forceinline__ void stage_strip(const SpmmArgs& a, int l0, uint8_t* strip) {
    if (a.src_rowmajor) {  // dense K x nlines row-major (spmm_int's B): strip[k][0..W) is a row slice
        const bool wv = (a.ldd % 4) == 0 && l0 + W <= a.nlines && (reinterpret_cast<uintptr_t>(a.dense) & 3) == 0;
        if (wv) {
            const int total = a.K * (W / 4);
            for (int e0 = threadIdx.x; e0 < total; e0 += 4 * NT) {
                uint32_t v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * NT;
                    v[u] = e < total ? *reinterpret_cast<const uint32_t*>(a.dense + (int64_t)(e / (W / 4)) * a.ldd + l0 +
                                                                          4 * (e % (W / 4)))
                                     : 0u;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * NT;
                    if (e < total) reinterpret_cast<uint32_t*>(strip)[e] = v[u];
                }
            }
        } else {
            for (int e = threadIdx.x; e < a.K * W; e += NT) {
                const int k = e / W, c = e % W;
                strip[e] = l0 + c < a.nlines ? (uint8_t)a.dense[(int64_t)k * a.ldd + l0 + c] : (uint8_t)0;
            }
        }
        return;
    }
    // W lines x K, K-major: 4 lines x 4 k per work item, 4x4 byte transpose, 4 items in flight
    const int total = ((a.K + 3) / 4) * (W / 4);
    for (int e0 = threadIdx.x; e0 < total; e0 += 4 * NT) {
        uint32_t r[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * NT;
            const int lg = e % (W / 4), k4 = e / (W / 4);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int l = l0 + lg * 4 + t;
                r[u][t] = (e < total && l < a.nlines)
                              ? *reinterpret_cast<const uint32_t*>(a.dense + (int64_t)l * a.ldd + 4 * k4)
                              : 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * NT;
            if (e >= total) break;
            const int lg = e % (W / 4), k4 = e / (W / 4);
            const uint32_t t0 = __byte_perm(r[u][0], r[u][1], 0x5140), t1 = __byte_perm(r[u][0], r[u][1], 0x7362);
            const uint32_t t2 = __byte_perm(r[u][2], r[u][3], 0x5140), t3 = __byte_perm(r[u][2], r[u][3], 0x7362);
            const uint32_t o[4] = {__byte_perm(t0, t2, 0x5410), __byte_perm(t0, t2, 0x7632),
                                   __byte_perm(t1, t3, 0x5410), __byte_perm(t1, t3, 0x7632)};
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (4 * k4 + t < a.K) *reinterpret_cast<uint32_t*>(strip + (size_t)(4 * k4 + t) * W + lg * 4) = o[t];
        }
    }
}

template <int W, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_spmm_strip(const SpmmArgs a) {
    extern __shared__ uint4 strip_raw[];
    uint8_t* strip = reinterpret_cast<uint8_t*>(strip_raw);
    // per-warp 32-row x W fp32 staging tile of the dr1 epilogue (row pitch kTileP
    // floats: conflict-free 16-byte lane accesses), so D_F is read and C written
    // with 8 rows x 64 bytes per instruction instead of 32 scattered rows
    float* tile = reinterpret_cast<float*>(strip + (((size_t)a.K * W + 15) & ~(size_t)15)) +
                  (threadIdx.x >> 5) * 32 * kTileP;
    XG_PDL_WAIT();
    if (a.run && !*a.run) return;
    if (a.bad && *a.bad) return;  // the build overflowed: the dense launch serves the call
    if (a.stamp && blockIdx.x == 0 && threadIdx.x == 0) a.stamp[0] = globaltimer_ns();
    constexpr int CH = NW * 32;  // sparse rows per item
    constexpr int NT = NW * 32;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nstrips = (a.nlines + W - 1) / W;
    const int nchunks = (a.nsp + CH - 1) / CH;
    const int items = nstrips * nchunks;
    const int i0 = (int)((int64_t)items * blockIdx.x / gridDim.x);
    const int i1 = (int)((int64_t)items * (blockIdx.x + 1) / gridDim.x);
    const uint32_t sbase = smem_u32(strip);
    // the dense lines' scale is one per-tensor value in the pipeline: its
    // float-float reciprocal is hoisted (per-line scales take the general form)
    const bool line_t = a.mode != kSpmmS32 && a.line_scale.stride == 0;
    const float2 lrc = line_t ? srcp(a.line_scale, 0) : make_float2(0.f, 0.f);
    int s = i0 / nchunks, ch = i0 % nchunks;  // current item (strip, chunk)
    int cur = -1;
    auto seg_at = [&](int chunk) {
        const int r = chunk * CH + w * 32 + lane;
        return r < a.nsp ? a.seg[r] : make_int2(0, 0);
    };
    // two-deep look-ahead: the segment of item it+2 and the first quad record
    // of item it+1 are in flight while item it runs
    auto first_rec = [&](int2 g) { return g.y > 0 ? __ldg(a.quad + g.x) : make_uint4(0u, 0u, 0u, 0u); };
    int2 sg_next = i0 < i1 ? seg_at(ch) : make_int2(0, 0);
    int2 sg_next2 = i0 + 1 < i1 ? seg_at(ch + 1 < nchunks ? ch + 1 : 0) : make_int2(0, 0);
    uint4 rec_next = first_rec(sg_next);
    for (int it = i0; it < i1; ++it) {
        if (s != cur) {
            __syncthreads();  // every warp is done with the previous strip
            stage_strip<W, NT>(a, s * W, strip);
            __syncthreads();
            cur = s;
        }
        const int r = ch * CH + w * 32 + lane;
        const int2 sg = sg_next;
        const uint4 rec0 = rec_next;
        const int s_item = s;
        if (++ch == nchunks) ch = 0, ++s;
        sg_next = sg_next2;
        rec_next = it + 1 < i1 ? first_rec(sg_next) : make_uint4(0u, 0u, 0u, 0u);
        sg_next2 = it + 2 < i1 ? seg_at(ch + 1 < nchunks ? ch + 1 : 0) : make_int2(0, 0);
        const int l0 = s_item * W;
        const bool vec = (a.ldo % 4) == 0 && l0 + W <= a.nlines;  // 16-byte rows of W columns
        // the epilogue's operand (D_F row slice / output column slice) in flight during the MACs
        const bool coop = a.mode == kSpmmRows && vec && W == 16;  // cooperative 8-row x 64 B accesses
        const int rq = lane & 3, rr0 = r - lane + (lane >> 2);  // rows rr0 + 8 i of the warp's 32
        float d[W];
        float4 g[4];
        if (coop) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int rr = rr0 + 8 * i;
                g[i] = rr < a.nsp ? *reinterpret_cast<const float4*>(a.din + (int64_t)rr * a.ldo + l0 + 4 * rq)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        } else if (r < a.nsp && a.mode == kSpmmRows) {
            const float* di = a.din + (int64_t)r * a.ldo + l0;
            if (vec) {
#pragma unroll
                for (int c = 0; c < W; c += 4) {
                    const float4 v = *reinterpret_cast<const float4*>(di + c);
                    d[c] = v.x; d[c + 1] = v.y; d[c + 2] = v.z; d[c + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int c = 0; c < W; ++c) d[c] = l0 + c < a.nlines ? di[c] : 0.0f;
            }
        } else if (r < a.nsp && a.mode == kSpmmColsT) {
#pragma unroll
            for (int c = 0; c < W; ++c) d[c] = l0 + c < a.nlines ? a.out[(int64_t)(l0 + c) * a.ldo + r] : 0.0f;
        }
        int acc[W];
#pragma unroll
        for (int c = 0; c < W; ++c) acc[c] = 0;
        // a row longer than kHeavyQ quads (e.g. a MinRule row with a zero statistic,
        // kept whole: sparse.cpp:55-60) is walked by the whole warp below instead
        const bool heavy = sg.y > kHeavyQ;
        const int nq = heavy ? 0 : sg.y;
        quads_mac<W>(a.quad, rec0, sg.x, nq, 1, sbase, acc);
        unsigned hm = __ballot_sync(0xffffffffu, heavy);
        while (hm) {
            const int src = __ffs(hm) - 1;
            hm &= hm - 1;
            const int hs = __shfl_sync(0xffffffffu, sg.x, src), hn = __shfl_sync(0xffffffffu, sg.y, src);
            int part[W];
#pragma unroll
            for (int c = 0; c < W; ++c) part[c] = 0;
            if (lane < hn) quads_mac<W>(a.quad, __ldg(a.quad + hs + lane), hs + lane, hn - lane, 32, sbase, part);
#pragma unroll
            for (int c = 0; c < W; ++c) {
                const int t = __reduce_add_sync(0xffffffffu, part[c]);
                if (lane == src) acc[c] += t;
            }
        }
        if (coop) {  // D_F rows of the warp: registers -> tile -> each lane's own row
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i)
                *reinterpret_cast<float4*>(tile + ((lane >> 2) + 8 * i) * kTileP + 4 * rq) = g[i];
            __syncwarp();
#pragma unroll
            for (int c = 0; c < W; c += 4) {
                const float4 v = *reinterpret_cast<const float4*>(tile + lane * kTileP + c);
                d[c] = v.x; d[c + 1] = v.y; d[c + 2] = v.z; d[c + 3] = v.w;
            }
        }
        if (r >= a.nsp && !coop) continue;
        if (a.mode == kSpmmS32) {  // C[r, l] (spmm_int)
            int32_t* o = a.out_s32 + (int64_t)r * a.ldo + l0;
            if (vec) {
#pragma unroll
                for (int c = 0; c < W; c += 4)
                    *reinterpret_cast<int4*>(o + c) = make_int4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
            } else {
#pragma unroll
                for (int c = 0; c < W; ++c)
                    if (l0 + c < a.nlines) o[c] = acc[c];
            }
            continue;
        }
        // deq(acc) = float(acc / (l_row * l_col)) (quantize.cpp:183), dr1: row = sparse row,
        // dr2: row = dense line (common.cuh dq_ff24, exact redo by dq_slow)
        const bool rows = a.mode == kSpmmRows;
        const int rs = min(r, a.nsp - 1);  // (a lane past the last row only helps the cooperative store)
        const float2 src_r = srcp(a.sp_scale, rs);
        float2 cc = make_float2(0.f, 0.f);
        if (line_t) cc = rows ? ff_mul(src_r, lrc) : ff_mul(lrc, src_r);
        uint32_t sm = 0;
        float t[W];
#pragma unroll
        for (int c = 0; c < W; ++c) {
            float2 cq = cc;
            if (!line_t) {
                const float2 lr = srcp(a.line_scale, min(l0 + c, a.nlines - 1));
                cq = rows ? ff_mul(src_r, lr) : ff_mul(lr, src_r);
            }
            t[c] = dq_ff24c(acc[c], cq, sm, 1u << c);
        }
        if (sm) {  // rare: exact redo of the flagged elements
#pragma unroll
            for (int c = 0; c < W; ++c)
                if ((sm >> c) & 1u) {
                    const int l = min(l0 + c, a.nlines - 1);
                    const float2 lr = srcp(a.line_scale, l);
                    const double ds = a.sp_scale.p[(int64_t)rs * a.sp_scale.stride];
                    const double dl = a.line_scale.p[(int64_t)l * a.line_scale.stride];
                    t[c] = rows ? dq_slow(acc[c], src_r, lr, ds, dl) : dq_slow(acc[c], lr, src_r, dl, ds);
                }
        }
        if (rows) {  // dr1: out[r, l] = fl(din[r, l] + deq) (pipeline.cpp:141-143)
            float* o = a.out + (int64_t)r * a.ldo + l0;
#pragma unroll
            for (int c = 0; c < W; ++c) d[c] = __fadd_rn(d[c], t[c]);
            if (coop) {  // each lane's row -> tile -> 8 rows x 64 bytes per store
#pragma unroll
                for (int c = 0; c < W; c += 4)
                    *reinterpret_cast<float4*>(tile + lane * kTileP + c) = make_float4(d[c], d[c + 1], d[c + 2], d[c + 3]);
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int rr = rr0 + 8 * i;
                    if (rr < a.nsp)
                        *reinterpret_cast<float4*>(a.out + (int64_t)rr * a.ldo + l0 + 4 * rq) =
                            *reinterpret_cast<const float4*>(tile + ((lane >> 2) + 8 * i) * kTileP + 4 * rq);
                }
            } else if (vec) {
#pragma unroll
                for (int c = 0; c < W; c += 4)
                    *reinterpret_cast<float4*>(o + c) = make_float4(d[c], d[c + 1], d[c + 2], d[c + 3]);
            } else {
#pragma unroll
                for (int c = 0; c < W; ++c)
                    if (l0 + c < a.nlines) o[c] = d[c];
            }
        } else {  // dr2, transposed: out[l, r] = fl(out + deq), then alpha/beta (pipeline.cpp:144-145, :195-202)
#pragma unroll
            for (int c = 0; c < W; ++c) {
                const int l = l0 + c;
                if (l >= a.nlines) break;
                float v = __fadd_rn(d[c], t[c]);
                if (a.has_c) {
                    v = __fadd_rn(__fmul_rn(a.alpha, v), __fmul_rn(a.beta, a.c_in[(int64_t)l * a.ldo + r]));
                } else if (a.alpha != 1.0f) {
                    v = __fmul_rn(v, a.alpha);
                }
                a.out[(int64_t)l * a.ldo + r] = v;
            }
        }
    }
    if (a.stamp_end) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(a.stamp_end, globaltimer_ns());
    }
}

// x[i, k] = non-zero uniform int8 in [-qmax, qmax] with probability `density`, else 0
// (a random sparse operand for the calibration; SplitMix64-style hash per element)
__global__ void k_random_masked_i8(int8_t* x, int rows, int cols, int64_t ld, uint32_t thr, int qmax,
                                   uint64_t seed) {
    const int64_t n = (int64_t)rows * ld;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (uint64_t)e * 0x9E3779B97F4A7C15ULL;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        const int c = (int)(e % ld);
        int v = 0;
        if (c < cols && (uint32_t)z < thr) {
            v = (int)((z >> 32) % (uint64_t)(2 * qmax)) - qmax;
            if (v >= 0) ++v;  // [-qmax, -1] u [1, qmax]
        }
        x[e] = (int8_t)v;
    }
}

int sm_count() {
    static const int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return n;
}

constexpr int kSpmmWarps = 16;

template <int W>
void launch_strip(const SpmmArgs& a, cudaStream_t s) {
    constexpr size_t kTileBytes = (size_t)kSpmmWarps * 32 * kTileP * 4;
    const size_t smem = (((size_t)a.K * W + 15) & ~(size_t)15) + kTileBytes;
    static bool attr = [] {
        cudaFuncSetAttribute(k_spmm_strip<W, kSpmmWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kSpmmSmemMax + kTileBytes));
        return true;
    }();
    (void)attr;
    const int nstrips = (a.nlines + W - 1) / W;
    const int nchunks = (a.nsp + kSpmmWarps * 32 - 1) / (kSpmmWarps * 32);
    const int64_t items = (int64_t)nstrips * nchunks;
    const int grid = (int)(items < sm_count() ? (items > 0 ? items : 1) : sm_count());
    k_spmm_strip<W, kSpmmWarps><<<grid, kSpmmWarps * 32, smem, s>>>(a);
}

}  // namespace

int spmm_strip_width(int K) {
    if ((size_t)K * 16 <= (size_t)kSpmmSmemMax) return 16;
    if ((size_t)K * 8 <= (size_t)kSpmmSmemMax) return 8;
    return 0;
}

void launch_qcsr_build(const int8_t* x, int rows, int cols, int64_t ld, const QCsr& q, const int* run, int* bad,
                       int max_quads, cudaStream_t s) {
    const int blocks = (rows + kBuildWarps - 1) / kBuildWarps;  // one warp per row, one atomic per block
    const int grid = blocks < 16 * sm_count() ? (blocks > 0 ? blocks : 1) : 16 * sm_count();
    k_qcsr_build<<<grid, kBuildWarps * 32, 0, s>>>(x, rows, cols, ld, q, run, bad, max_quads);
}

void launch_qcsr_from_csr(const int32_t* rp, const int32_t* ci, const int8_t* v, int rows, const QCsr& q,
                          cudaStream_t s) {
    const int blocks = (rows + kBuildWarps * kBuildRows - 1) / (kBuildWarps * kBuildRows);
    const int grid = blocks < 4 * sm_count() ? (blocks > 0 ? blocks : 1) : 4 * sm_count();
    k_qcsr_from_csr<<<grid, kBuildWarps * 32, 0, s>>>(rp, ci, v, rows, q);
}

void launch_random_masked_i8(int8_t* x, int rows, int cols, int64_t ld, double density, int qmax, uint64_t seed,
                             cudaStream_t s) {
    const double t = density * 4294967296.0;
    const uint32_t thr = t >= 4294967295.0 ? 0xffffffffu : (uint32_t)t;
    k_random_masked_i8<<<4 * sm_count(), 256, 0, s>>>(x, rows, cols, ld, thr, qmax, seed);
}

bool launch_spmm_strip(const SpmmArgs& a, cudaStream_t s) {
    const int W = spmm_strip_width(a.K);
    if (W == 16) launch_strip<16>(a, s);
    else if (W == 8) launch_strip<8>(a, s);
    else return false;
    return true;
}

}  // namespace xg
