// Internal host-side launch interfaces shared by the .cu translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace xg {

// Device-resident scalars of one pipeline run.  Zeroed at the start of a run;
// every field is written by kernels only, read back once at the end.
struct DevScalars {
    uint32_t maxA, maxB;      // float bits of max|A|, max|B| (matrix.cpp:51-58)
    uint32_t maxRA, maxRB;    // float bits of max|RA|, max|RB|
    uint32_t retA, retB;      // float bits of max retained |a|, |b| (sparse.cpp:200-203)
    int nonfinite;            // any non-finite input seen
    int sel;                  // 1 -> sparse compensation path
    unsigned long long nnzA, nnzB;
    int nflag;                // AvgRule statistics needing the exact sequential sum
    int pad0;
    double lamA, lamB;        // per-tensor scales (PerTensor scheme)
    double lamRA, lamRB;      // residual per-tensor scales (pipeline.cpp:86-93)
    double lamAred, lamBred;  // per-tensor scales of the reduced operands
    double densA, densB;
    int path;
    int pad1;
    // float-float reciprocals (common.cuh: ff_recip) of the per-tensor scales above,
    // written next to them so the GEMM epilogues do no fp64 division
    float2 rA, rB, rRA, rRB, rAred, rBred;
    // %globaltimer stamps of the graph path's stage boundaries (ns): pipeline
    // start, D_F GEMM begin / end, compensation begin / end; 0 = not written
    unsigned long long ts[5];
    unsigned done;  // CTAs of the compensation GEMM finished (the last one writes the report)
    unsigned pad2;
    // sparse compensation on CUDA cores (spmm.cu) instead of the masked-dense
    // tensor-core launch: chosen by k_dispatch from the cost model; csr_bad is
    // raised by the CSR build (capacity / a very long row), the dense launch
    // then serves the call
    int csr, csr_bad;
    unsigned long long qcurA, qcurB;  // quads handed out by the two CSR builds
};

// Cost model of the compensation choice (k_dispatch): masked-dense tcgen05
// t_d = 4MNK / p_tc against the CUDA-core CSR path t_c = max((nnzA N + nnzB M)
// / p_sp, MN c_el) + 3 (M + N) K / bw (the CSR builds), c_el the per-output-element
// cost of its two exact epilogue passes.  The CSR path is taken when t_c <
// 0.9 t_d.  Rates measured on B200 (xg_calibrate_eta re-measures p_tc, p_sp).
// force: 0 auto, 1 dense, 2 CSR.
struct CompModel {
    double p_tc, p_sp, bw, c_el;
    int force;
    int csr_ok;  // host: the CSR path is available for this shape (strip fits, buffers allocated)
};
const CompModel& comp_model();
void set_comp_model(const CompModel& m);

struct QuantRowsArgs {
    const float* x;
    int rows, cols;
    int64_t ld;
    int bits, rounding;
    int per_row;            // 1: PerRow scales computed here; 0: per-tensor from *tensor_max
    const uint32_t* tensor_max;  // float bits (per-tensor)
    double* lam_out;        // [rows] (per_row) — may be null
    float2* rcp_out;        // [rows] ff_recip(lam) next to lam_out — may be null
    int8_t* q;              // [rows x ldq]
    int64_t ldq;
    uint32_t* gmax;         // atomicMax of max|x| (float bits), may be null
    uint32_t* rmax;         // atomicMax of max|x - deq| (float bits), may be null
    int* nonfinite;
};

struct QuantColsArgs {
    const float* x;          // rows(K) x cols(N) row-major
    int rows, cols;
    int64_t ld;
    int bits, rounding;
    int per_col;
    const uint32_t* colmax;  // float bits [cols] (per_col)
    const uint32_t* tensor_max;
    double* lam_out;         // [cols] (per_col)
    float2* rcp_out;         // [cols] ff_recip(lam) next to lam_out — may be null
    int8_t* qT;              // [cols x ldq] transposed (K-major)
    int64_t ldq;
    uint32_t* rmax;
    const int* nonfinite;    // see SelectArgs::nonfinite (set by the column absmax pass)
};

// K3: residual quantisation + threshold selection of the original operand.
struct SelectArgs {
    const float* x;
    int rows, cols;          // A: M x K ; B: K x N
    int64_t ld;
    int bits, rounding;
    int vec;                 // 1: per-row (A) / per-col (B) scales in lam; 0: per-tensor
    const double* lam;       // [rows] (A) / [cols] (B)
    const uint32_t* tensor_max;  // float bits of max|X| for the per-tensor scale
    const uint32_t* rmax;    // float bits of max|R| -> lambda_R
    int do_select;
    const float* stat;       // row stats (A) / column stats (B)
    double thr_m;
    int policy;
    const uint32_t* other_max;  // float bits of max|other operand| (MinRule scale_other)
    int8_t* rq;              // residual ints (A: rows x ldq; B: transposed cols x ldq)
    int8_t* red;             // reduced operand ints (same layout), null if !do_select
    int64_t ldq;
    unsigned long long* nnz;
    uint32_t* retmax;
    // fix-up mode: rewrite `red` with the retained-max scale when it differs
    int fix_mode;
    // set by the K1 kernels when an input is not finite: the call will fail
    // (pipeline.cpp:50-52), so the table-driven kernels exit instead of
    // indexing their dequant tables with NaN bit patterns
    const int* nonfinite;
    // stage dump only (null otherwise): kept-element bitmask, bit (c % 32) of
    // word [r * keep_ld + c / 32] for row r of the operand as laid out above
    // (A: row i over k; B: row j of B^T over k), OR-ed in by the kernel
    uint32_t* keep;
    int64_t keep_ld;
};

void launch_absmax_global(const float* x, int64_t n, uint32_t* gmax, int* nonfinite,
                          cudaStream_t s);
void launch_absmax_cols(const float* x, int rows, int cols, int64_t ld, uint32_t* colmax,
                        uint32_t* gmax, int* nonfinite, cudaStream_t s);
void launch_quant_rows(const QuantRowsArgs& a, cudaStream_t s);
void launch_quant_cols_T(const QuantColsArgs& a, cudaStream_t s);
// column maxima + quantisation of B in one DRAM pass (VectorWise, nearest);
// false when not applicable (then absmax_cols + quant_cols_T)
bool launch_quant_cols_fused(const QuantColsArgs& a, uint32_t* gmax, int* nonfinite, cudaStream_t s);
void launch_select_rows(const SelectArgs& a, cudaStream_t s);
void launch_select_cols_T(const SelectArgs& a, cudaStream_t s);
void launch_lambdas(DevScalars* sc, int bits, cudaStream_t s);
void launch_dispatch(DevScalars* sc, int bits, int64_t MK, int64_t KN, double density_limit,
                     int reduce, cudaStream_t s, int M = 0, int N = 0, int K = 0, int csr_ok = 0,
                     const CompModel* model = nullptr);

// statistics over D_F (pipeline.cpp:215-247)
// Deferred exact-mean fallback (AvgRule): the operands whose selection the
// statistics drive (A rows: M x inner, B columns: inner x N) and the threshold
// multiplier; `widen` (test hook) scales the verified-rounding interval by
// 2^widen so the deferred path is exercised on every statistic.
struct StatsDefer {
    const float* a;
    int64_t lda;
    const float* b;
    int64_t ldb;
    int inner;
    double thr_m;
    int widen;
    // row-sharded pipeline: column statistics that need the exact sequential
    // sum are listed here (they span other ranks) instead of computed locally
    int* remote_cols;
    int* n_remote;
    int remote_cap;
};
void launch_stats(const float* d, int rows, int cols, int policy, float* row_stat,
                  float* col_stat, double* row_sum, double* col_sum, int* flags, int* nflag,
                  cudaStream_t s, const StatsDefer* def = nullptr);
// zero the device scalars / column maxima and initialise the statistics accumulators
void launch_pipe_init(void* sc, int sc_bytes, uint32_t* colmax, int N, double* rsum, double* csum,
                      float* rstat, float* cstat, int M, int policy, int reduce, cudaStream_t s,
                      unsigned long long* ts0 = nullptr);
// the two halves of launch_stats, split around the row-sharded column reduction
// mode 0: initialise + accumulate; 1: initialise only; 2: accumulate only (row
// pointers offset to a row chunk, column accumulators shared by all chunks)
void launch_stats_partial(const float* d, int rows, int cols, int policy, float* row_stat,
                          float* col_stat, double* row_sum, double* col_sum, int* nflag, cudaStream_t s,
                          int mode = 0);
void launch_stats_final(const float* d, int rows, int cols, int col_n, int policy, float* row_stat,
                        float* col_stat, double* row_sum, double* col_sum, int* flags, int* nflag,
                        cudaStream_t s, const StatsDefer* def);
void launch_pack_remote_cols(const float* d, int rows, int cols, const int* list, const int* n, int cap,
                             int mpad, float* buf, cudaStream_t s);
void launch_remote_col_means(const float* gath, int g, const int* rank_rows, int mpad, int cap,
                             const int* list, const int* n, int col_n, float* col_stat, cudaStream_t s);

void fill_u32(uint32_t* p, uint32_t v, int64_t n, cudaStream_t s);

}  // namespace xg
