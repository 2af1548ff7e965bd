// Host-side planning/launch of the tcgen05 GEMM (gemm.cuh).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm_types.h"

namespace sf {
namespace gemm {

struct Op {
  CUtensorMap ta;
  CUtensorMap tb;
  Params p;
  dim3 grid;
  size_t smem;
};

// Encode a 2-D K-major bf16 tensor map (rows x K, row stride `ld` elements)
// with a 64 x box_rows SWIZZLE_128B box.
int make_map(CUtensorMap* m, const void* ptr, int rows, int K, int ld, int box_rows);

// Plan one GEMM. `A` has rows_a rows, `B` rows_b rows, both K-major with K
// columns (row strides lda/ldb elements). splits=0 picks split-K so that the
// grid covers ~`target_ctas` CTAs. ws/counters may be null when splits == 1.
int plan(Op* op, const void* A, int rows_a, int lda, const void* B, int rows_b, int ldb, int K,
         int bn, int splits, int swap_ab, const EpiArgs& e, float* ws, size_t ws_bytes,
         int* counters, int n_counters, int max_stages = 8);

int launch(const Op& op, cudaStream_t stream, bool pdl);

// split-K workspace needed for a plan (bytes) and counters (ints)
size_t ws_bytes_needed(int rows_a, int rows_b, int K, int bn, int splits);

}  // namespace gemm
}  // namespace sf
