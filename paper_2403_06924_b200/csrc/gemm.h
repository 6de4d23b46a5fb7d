// Host interface of the tcgen05 INT8 GEMM (gemm_tc.cuh).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace xg {

struct GemmArgs;

// rows x K int8 operand, K-major, row pitch `ld` bytes (multiple of 16).
struct KOperand {
    const int8_t* p;
    int rows;
    int64_t ld;
};

// 2-D fp32 tensor map (rows x cols, row pitch ld floats), box box_cols x box_rows,
// no swizzle, zero fill.  Returns false if the layout is not TMA-compatible.
bool make_tmap_f32(void* tmap /* CUtensorMap* */, const float* p, int rows, int cols, int64_t ld,
                   int box_cols, int box_rows);

// Launches the persistent GEMM with epilogue `epi` (EpiMode).  ops[i] becomes
// tensor map i; is_b[i] selects the B-operand box height.
void gemm_i8(int epi, const KOperand* ops, const int* is_b, int nops, const GemmArgs& args,
             cudaStream_t s);

// Both pipeline GEMMs of an M x N problem run the pair kernel (whose
// %globaltimer stamps give the report's stage times).
bool pair_gemm_used(int M, int N);

}  // namespace xg
