// Shared host/device definitions of the tcgen05 GEMM (kernels in gemm.cuh).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace sf {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kEpiWarps = 8;                        // 2 per TMEM lane quarter
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kThreads = 64 + kEpiThreads;          // warp 0 TMA, warp 1 MMA, 8 epilogue warps
constexpr uint32_t kAStageBytes = BM * BK * 2;
constexpr int kMaxSplits = 16;                      // cluster size along the split-K axis

enum EpiKind : int {
  EPI_F32 = 0,        // out_f32[m, n] = acc * r[m] (+ bias[n])
  EPI_BF16 = 1,       // out_bf16[m, n] = bf16(acc * r[m] (+ bias[n]))
  EPI_QKV = 2,        // RMS scale, RoPE on q/k (paired rows), q/k row-major, v transposed
  EPI_RESID = 3,      // x[m, n] += acc; xb = bf16(x); ssq partials per 128-feature group
  EPI_GEGLU = 4,      // RMS scale, h[m, n/2] = gelu_tanh(gate) * up for paired rows
  EPI_TANH_BF16 = 5,  // out_bf16[m, n] = bf16(tanh(acc + bias[n]))  (draft MLP hidden)
  EPI_KINDS = 6
};

struct EpiArgs {
  int kind;
  int M;  // valid token rows
  int N;  // valid output features
  float* out_f32;
  int ld_f32;
  __nv_bfloat16* out_bf16;
  int ld_bf16;
  const float* bias;  // per output feature (F32 / BF16 / TANH), may be null
  // RMSNorm row scale r[m] = rsqrt(sum_g ssq_in[g * ssq_ld + m] * inv_width + eps)
  const float* ssq_in;
  int ssq_groups;
  int ssq_ld;
  float inv_width;
  float eps;
  // QKV
  __nv_bfloat16* q;
  __nv_bfloat16* k;
  __nv_bfloat16* vt;
  int vt_ld;
  const float2* rope;  // [head_dim/2][rope_ld] (cos, sin): position fastest
  int rope_ld;
  int q_features;      // q_heads * head_dim
  int env_rows, seg_len, pos0;
  // RESID (x, xb are [M, N] row-major)
  float* x;
  __nv_bfloat16* xb;
  float* ssq_out;
  int ssq_out_ld;
};

struct Params {
  int rows_a, rows_b, K;
  int bn;
  int num_kb, kb_per_split, splits;
  int stages;
  int swap_ab;
  int tiles_a, tiles_b, total_tiles;
  uint32_t smem_stage_region;  // bytes reserved for the TMA ring (>= split-K staging)
  unsigned long long* dbg;     // optional %globaltimer stamps of CTA (0,0,0) (null: off)
  float* ws;                   // split-K partials [split][tile][chunk][4][128][4] (swap, S > 1)
  // optional live row count on the device (compacted bucket bodies of the
  // replanning graph): rows = min(rows_a, *rows_dev * rows_mul); row tiles
  // past it are not visited (batched kernels only; null: rows_a)
  const int* rows_dev;
  int rows_mul;
  EpiArgs e;
};

}  // namespace gemm
}  // namespace sf
