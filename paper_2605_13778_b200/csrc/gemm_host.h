// Host-side planning/launch of the tcgen05 GEMMs (gemm.cuh).
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
  int cluster = 1;   // split-K cluster size (swap kernel) / 2 for CTA pairs
  bool pair = false;  // batched GEMM on 2-SM CTA pairs (gemm_pair_kernel)
  size_t smem = 0;
  size_t ws_bytes = 0;  // split-K workspace the caller must attach as p.ws
  void* fn = nullptr;  // specialised kernel
};

// Encode a 2-D K-major bf16 tensor map (rows x K, row stride `ld` elements)
// with a 64 x box_rows SWIZZLE_128B box.
int make_map(CUtensorMap* m, const void* ptr, int rows, int K, int ld, int box_rows);

// Number of K splits that spreads `tiles` output tiles over the SMs.
int auto_splits(int tiles, int num_kb);

// Plan one GEMM. swap_ab=1: A rows are output features (weights), B rows are
// token rows, bn covers the tokens, split-K through a CTA cluster (splits<=0:
// auto). swap_ab=0: A rows are token rows, B rows are features, persistent
// whole-K tiles (splits ignored).
int plan(Op* op, const void* A, int rows_a, int lda, const void* B, int rows_b, int ldb, int K,
         int bn, int splits, int swap_ab, const EpiArgs& e, int max_stages = 8);

int launch(const Op& op, cudaStream_t stream, bool pdl);

}  // namespace gemm
}  // namespace sf
