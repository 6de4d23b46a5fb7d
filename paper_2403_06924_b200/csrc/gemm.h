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

// Launches the persistent GEMM with epilogue `epi` (EpiMode).  ops[i] becomes
// tensor map i; is_b[i] selects the B-operand box height.
void gemm_i8(int epi, const KOperand* ops, const int* is_b, int nops, const GemmArgs& args,
             cudaStream_t s);

}  // namespace xg
