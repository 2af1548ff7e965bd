// tcgen05 GEMM for the pi0-scale Action Expert (sm_100a).
//
//   D[a, b] = sum_k A[a, k] * B[b, k]      (A, B bf16 K-major; fp32 accumulation in TMEM)
//
// One CTA computes a 128 x BN tile (UMMA M=128, N=BN<=256, K=16 per
// instruction) over a K range; warp 0 is the TMA producer (SWIZZLE_128B tiles
// 64 elements deep into a `stages`-deep mbarrier ring), warp 1 allocates TMEM
// and issues tcgen05.mma from one elected lane, warps 2-5 are the epilogue
// (tcgen05.ld 32x32b -> registers -> fused op -> global).
//
// Two orientations share the kernel:
//  * swap-AB (batch-1 rounds, 51..416 token rows): A = weights, so the 128
//    TMEM lanes are output features and the BN columns are token rows. Weight
//    tiles fill the M=128 slot; split-K spreads the weight stream over all
//    148 SMs; partials are reduced deterministically by the last-arriving CTA
//    of each tile (fixed split order), which then runs the fused epilogue.
//  * normal (batched envs): A = token rows, B = weights, BN = 256 features.
// PDL: weight tiles do not depend on the previous kernel, so the producer
// issues them BEFORE griddepcontrol.wait; only activation tiles wait.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "sm100.cuh"
#include "gemm_types.h"

namespace sf {
namespace gemm {

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanhf(k0 * (x + k1 * x * x * x)));
}

__device__ __forceinline__ float row_scale(const EpiArgs& e, int m) {
  if (!e.ssq_in) return 1.0f;
  float s = 0.f;
  for (int g = 0; g < e.ssq_groups; ++g) s += e.ssq_in[g * e.ssq_ld + m];
  return rsqrtf(s * e.inv_width + e.eps);
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Apply the fused op to one 16-column chunk held by this thread.
// swap: lane_row = feature, columns = tokens; else lane_row = token, columns = features.
__device__ __forceinline__ void apply_chunk(const Params& p, float (&v)[16], int lane_row, int c0,
                                            const float* rs_cols, float rs_row, float* red_q,
                                            float& ssq_acc) {
  const EpiArgs& e = p.e;
  const bool swap = p.swap_ab;
  const int tile_a = blockIdx.x, tile_b = blockIdx.y;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int m = swap ? tile_b * p.bn + c0 + j : tile_a * BM + lane_row;
    const float r = swap ? rs_cols[c0 + j] : rs_row;
    if (e.kind != EPI_RESID) v[j] *= r;
  }
  switch (e.kind) {
    case EPI_F32:
    case EPI_BF16:
    case EPI_TANH_BF16: {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = swap ? tile_b * p.bn + c0 + j : tile_a * BM + lane_row;
        const int n = swap ? tile_a * BM + lane_row : tile_b * p.bn + c0 + j;
        if (m < e.M && n < e.N) {
          float o = e.bias ? v[j] + e.bias[n] : v[j];
          if (e.kind == EPI_TANH_BF16) o = tanhf(o);
          if (e.kind == EPI_F32) e.out_f32[(size_t)m * e.ld_f32 + n] = o;
          else e.out_bf16[(size_t)m * e.ld_bf16 + n] = __float2bfloat16_rn(o);
        }
      }
      break;
    }
    case EPI_GEGLU:
    case EPI_QKV: {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float partner = swap ? __shfl_xor_sync(0xffffffffu, v[j], 1) : v[j ^ 1];
        const int m = swap ? tile_b * p.bn + c0 + j : tile_a * BM + lane_row;
        const int n = swap ? tile_a * BM + lane_row : tile_b * p.bn + c0 + j;
        if (m >= e.M || n >= e.N) continue;
        const int second = n & 1;
        if (e.kind == EPI_GEGLU) {
          // device rows interleave (gate_i, up_i) -> h_i = gelu(gate_i) * up_i
          if (!second)
            e.out_bf16[(size_t)m * e.ld_bf16 + (n >> 1)] =
                __float2bfloat16_rn(gelu_tanh(v[j]) * partner);
        } else if (n < e.q_features + 256) {
          // rows (2i, 2i+1) = (dim i, dim i+128) of one head: rotate_half RoPE
          const int local = m % e.env_rows;
          const int pos = e.pos0 + (local % e.seg_len);
          const int i = (n & 255) >> 1;
          const float2 cs = e.rope[pos * 128 + i];
          const float a = second ? partner : v[j];
          const float b = second ? v[j] : partner;
          const float y = second ? (b * cs.x + a * cs.y) : (a * cs.x - b * cs.y);
          const int dim = i + (second << 7);
          if (n < e.q_features)
            e.q[(size_t)m * e.q_features + (n & ~255) + dim] = __float2bfloat16_rn(y);
          else
            e.k[(size_t)m * 256 + dim] = __float2bfloat16_rn(y);
        } else {
          const int d = n - e.q_features - 256;
          e.vt[(size_t)d * e.vt_ld + m] = __float2bfloat16_rn(v[j]);
        }
      }
      break;
    }
    case EPI_RESID: {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = swap ? tile_b * p.bn + c0 + j : tile_a * BM + lane_row;
        const int n = swap ? tile_a * BM + lane_row : tile_b * p.bn + c0 + j;
        float sq = 0.f;
        if (m < e.M && n < e.N) {
          const size_t o = (size_t)m * e.N + n;
          const float xn = e.x[o] + v[j];
          e.x[o] = xn;
          e.xb[o] = __float2bfloat16_rn(xn);
          sq = xn * xn;
        }
        if (swap) {
          // sum over the 128 features (lanes of 4 warps) of this token column
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
          if ((threadIdx.x & 31) == 0) red_q[c0 + j] = sq;
        } else {
          ssq_acc += sq;
        }
      }
      break;
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t b_bytes = (uint32_t)p.bn * BK * 2;
  const uint32_t stage_bytes = kAStageBytes + ((b_bytes + 1023) & ~1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* tmem_full = empty + p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  float* rs_cols = reinterpret_cast<float*>(tmem_slot + 4);  // [256]
  float* red = rs_cols + 256;                                 // [4][256]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_a = blockIdx.x, tile_b = blockIdx.y, split = blockIdx.z;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kb_per_split, p.num_kb - kb0);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(tmem_full, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (sm100::elect_one()) {
      sm100::tma_prefetch_desc(&tma_a);
      sm100::tma_prefetch_desc(&tma_b);
      const uint64_t pol_w = sm100::policy_evict_first();
      const uint64_t pol_x = sm100::policy_evict_last();
      const CUtensorMap* tw = p.swap_ab ? &tma_a : &tma_b;  // weights
      const CUtensorMap* tx = p.swap_ab ? &tma_b : &tma_a;  // activations
      const int w_row = p.swap_ab ? tile_a * BM : tile_b * p.bn;
      const int x_row = p.swap_ab ? tile_b * p.bn : tile_a * BM;
      const uint32_t w_off = p.swap_ab ? 0 : kAStageBytes;
      const uint32_t x_off = p.swap_ab ? kAStageBytes : 0;
      const int pre = min(p.stages, nkb);
      // weights first: independent of the previous kernel (PDL overlap)
      for (int i = 0; i < pre; ++i) {
        uint8_t* st = smem + i * stage_bytes;
        sm100::mbar_arrive_expect_tx(&full[i], kAStageBytes + b_bytes);
        sm100::tma_load_2d(tw, &full[i], st + w_off, (kb0 + i) * BK, w_row, pol_w);
      }
      sm100::pdl_wait();
      for (int i = 0; i < pre; ++i)
        sm100::tma_load_2d(tx, &full[i], smem + i * stage_bytes + x_off, (kb0 + i) * BK, x_row, pol_x);
      for (int i = pre; i < nkb; ++i) {
        const int s = i % p.stages;
        sm100::mbar_wait(&empty[s], ((i / p.stages) & 1) ^ 1);
        uint8_t* st = smem + s * stage_bytes;
        sm100::mbar_arrive_expect_tx(&full[s], kAStageBytes + b_bytes);
        sm100::tma_load_2d(tw, &full[s], st + w_off, (kb0 + i) * BK, w_row, pol_w);
        sm100::tma_load_2d(tx, &full[s], st + x_off, (kb0 + i) * BK, x_row, pol_x);
      }
    }
  } else if (warp == 1) {
    if (sm100::elect_one()) {
      const uint32_t idesc = sm100::make_idesc_bf16(BM, p.bn);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % p.stages;
        sm100::mbar_wait(&full[s], (i / p.stages) & 1);
        sm100::tc_fence_after();
        const uint32_t a_addr = sm100::smem_u32(smem + s * stage_bytes);
        const uint32_t b_addr = a_addr + kAStageBytes;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          sm100::umma_bf16(tmem, sm100::make_sw128_desc(a_addr + k * 32),
                           sm100::make_sw128_desc(b_addr + k * 32), idesc, (i | k) != 0);
        }
        sm100::umma_commit(&empty[s]);
      }
      sm100::umma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int et = threadIdx.x - 64;  // 0..127
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int lane_row = q * 32 + lane;
    const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
    sm100::pdl_wait();
    if (et == 0) sm100::pdl_launch_dependents();
    sm100::mbar_wait(tmem_full, 0);
    sm100::tc_fence_after();
    const int tiles = p.tiles_a * p.tiles_b;
    const int tile_id = tile_a * p.tiles_b + tile_b;
    bool proceed = true;
    if (p.splits > 1) {
      float* mine = p.ws + ((size_t)split * tiles + tile_id) * p.bn * BM;
      for (int c0 = 0; c0 < p.bn; c0 += 16) {
        uint32_t r[16];
        sm100::tmem_ld16(t_lane + c0, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) mine[(size_t)(c0 + j) * BM + lane_row] = __uint_as_float(r[j]);
      }
      __threadfence();
      epi_bar();
      if (et == 0) {
        const int prev = atomicAdd(&p.counters[tile_id], 1);
        const int last = prev == p.splits - 1;
        if (last) p.counters[tile_id] = 0;  // re-arm for the next launch / graph replay
        *last_flag = last;
      }
      epi_bar();
      proceed = *last_flag != 0;
      if (proceed) __threadfence();
    }
    if (proceed) {
      const EpiArgs& e = p.e;
      float rs_row = 1.f;
      if (p.swap_ab) {
        for (int c = et; c < p.bn; c += 128) {
          const int m = tile_b * p.bn + c;
          rs_cols[c] = (e.kind != EPI_RESID && m < e.M) ? row_scale(e, m) : 1.f;
        }
        epi_bar();
      } else {
        const int m = tile_a * BM + lane_row;
        rs_row = (e.kind != EPI_RESID && m < e.M) ? row_scale(e, m) : 1.f;
      }
      float ssq_acc = 0.f;
      for (int c0 = 0; c0 < p.bn; c0 += 16) {
        uint32_t r[16];
        sm100::tmem_ld16(t_lane + c0, r);
        sm100::tmem_ld_wait();
        float v[16];
        if (p.splits > 1) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
          for (int s = 0; s < p.splits; ++s) {
            if (s == split) {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] += __uint_as_float(r[j]);
            } else {
              const float* part = p.ws + ((size_t)s * tiles + tile_id) * p.bn * BM;
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] += __ldcg(part + (size_t)(c0 + j) * BM + lane_row);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
        }
        apply_chunk(p, v, lane_row, c0, rs_cols, rs_row, red + q * 256, ssq_acc);
        if (e.kind == EPI_RESID && !p.swap_ab && ((c0 + 16) % 128 == 0 || c0 + 16 >= p.bn)) {
          const int m = tile_a * BM + lane_row;
          const int g = (tile_b * p.bn + c0) / 128;
          if (m < e.M) e.ssq_out[(size_t)g * e.ssq_out_ld + m] = ssq_acc;
          ssq_acc = 0.f;
        }
      }
      if (e.kind == EPI_RESID && p.swap_ab) {
        epi_bar();
        const int g = (tile_a * BM) / 128;
        for (int c = et; c < p.bn; c += 128) {
          const int m = tile_b * p.bn + c;
          if (m < e.M)
            e.ssq_out[(size_t)g * e.ssq_out_ld + m] =
                ((red[c] + red[256 + c]) + red[512 + c]) + red[768 + c];
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<kTmemCols>(tmem);
  }
}

}  // namespace gemm
}  // namespace sf
