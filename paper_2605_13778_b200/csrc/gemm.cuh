// tcgen05 GEMM for the pi0-scale Action Expert (sm_100a).
//
//   D[a, b] = sum_k A[a, k] * B[b, k]   (A, B bf16 K-major; fp32 accumulation in TMEM)
//
// Warp roles (320 threads): warp 0 = TMA producer (SWIZZLE_128B 64-deep
// K tiles into a `stages`-deep mbarrier ring), warp 1 = TMEM allocator + MMA
// issuer (one elected lane, UMMA 128 x BN x 16), warps 2-9 = epilogue
// (tcgen05.ld 32x32b; two warps per TMEM lane quarter split the columns).
// Epilogues are compile-time specialised per fused op (RMS scale + RoPE,
// residual + RMS partials, GeGLU, tanh, plain store) with vectorised stores.
//
// Two kernels:
//  * gemm_swap_kernel (batch-1 shapes, <= 256 token rows): A = weights, so the
//    128 TMEM lanes are output features and BN columns are token rows; split-K
//    spreads the weight stream over up to 148 SMs. The S split CTAs of a tile
//    form a thread-block cluster: each stages its fp32 partial in SMEM, then
//    every CTA reduces 1/S of the columns over DSMEM in a fixed split order
//    (deterministic) and runs the fused epilogue on them. No global workspace,
//    no serial last-CTA reduction.
//  * gemm_persistent_kernel (batched envs): A = token rows, B = weights,
//    BN = 256; one CTA per SM walks tiles (features fastest, so a row tile's
//    activations are shared through L2); two TMEM accumulators (512 columns)
//    let the epilogue of tile i overlap the MMAs of tile i+1.
// PDL: weight tiles do not depend on the previous kernel, so the producer
// issues them BEFORE griddepcontrol.wait; activation tiles wait.
#pragma once

#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm_types.h"
#include "sm100.cuh"

namespace sf {
namespace gemm {

namespace cg = cooperative_groups;

// MUFU tanh (max rel. error ~2^-11): its result feeds a bf16 rounding, so the
// approximation is invisible at the stored precision.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanh_fast(k0 * (x + k1 * x * x * x)));
}

__device__ __forceinline__ float row_scale(const EpiArgs& e, int m) {
  if (!e.ssq_in) return 1.0f;
  float s = 0.f;
  for (int g = 0; g < e.ssq_groups; ++g) s += __ldcg(e.ssq_in + g * e.ssq_ld + m);
  return rsqrtf(s * e.inv_width + e.eps);
}

__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// Residual rows of one 16-column chunk in the staged layout (lane: row
// pass * 16 + lane / 2, columns 8 (lane & 1) .. +8): two 32 B loads per lane.
__device__ __forceinline__ void resid_load(const float* x, int M, int N, int m0w, int n0, int lane,
                                           float (&xo)[2][8]) {
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const int row = m0w + pass * 16 + (lane >> 1);
    if (row < M) {
      asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(xo[pass][0]), "=f"(xo[pass][1]), "=f"(xo[pass][2]), "=f"(xo[pass][3]),
                     "=f"(xo[pass][4]), "=f"(xo[pass][5]), "=f"(xo[pass][6]), "=f"(xo[pass][7])
                   : "l"(x + (size_t)row * N + n0 + (lane & 1) * 8));
    } else {
#pragma unroll
      for (int z = 0; z < 8; ++z) xo[pass][z] = 0.f;
    }
  }
}
// 32-byte global store (one STG.256: a full L2 sector per lane)
__device__ __forceinline__ void st_global_v8(void* p, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
               "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

// ------------------------------------------------------------- epilogues
//
// SWAP: thread = feature n (fixed), columns = tokens m0 + j.
template <int KIND>
__device__ __forceinline__ void epi_swap(const EpiArgs& e, int n, int m0, const float (&v)[16],
                                         const float* rs, float* red_q, int c0) {
  const bool nvalid = n < e.N;
  if (KIND == EPI_F32 || KIND == EPI_BF16 || KIND == EPI_TANH_BF16) {
    const float b = (e.bias && nvalid) ? e.bias[n] : 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int m = m0 + j;
      if (nvalid && m < e.M) {
        float o = v[j] * rs[c0 + j] + b;
        if (KIND == EPI_TANH_BF16) o = tanh_fast(o);
        if (KIND == EPI_F32) e.out_f32[(size_t)m * e.ld_f32 + n] = o;
        else e.out_bf16[(size_t)m * e.ld_bf16 + n] = __float2bfloat16_rn(o);
      }
    }
  } else if (KIND == EPI_GEGLU) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float x = v[j] * rs[c0 + j];
      const float partner = __shfl_xor_sync(0xffffffffu, x, 1);
      const int m = m0 + j;
      if (nvalid && m < e.M && !(n & 1))
        e.out_bf16[(size_t)m * e.ld_bf16 + (n >> 1)] = __float2bfloat16_rn(gelu_tanh(x) * partner);
    }
  } else if (KIND == EPI_QKV) {
    if (n < e.q_features + 256) {
      const int second = n & 1;
      const int i = (n & 255) >> 1;
      const int dim = i + (second << 7);
      // all 16 (cos, sin) loads in flight before any store (stores could
      // alias the table in the compiler's view and would serialise them)
      float2 csv[16];
      {
        int local = m0 % e.env_rows;
        int t = local % e.seg_len;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          csv[j] = __ldg(e.rope + (size_t)i * e.rope_ld + e.pos0 + t);
          if (++local == e.env_rows) local = 0, t = -1;
          if (++t == e.seg_len) t = 0;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float x = v[j] * rs[c0 + j];
        const float partner = __shfl_xor_sync(0xffffffffu, x, 1);
        const int m = m0 + j;
        if (!nvalid || m >= e.M) continue;
        const float2 cs = csv[j];
        const float a = second ? partner : x;
        const float b = second ? x : partner;
        const float y = second ? (b * cs.x + a * cs.y) : (a * cs.x - b * cs.y);
        if (n < e.q_features) e.q[(size_t)m * e.q_features + (n & ~255) + dim] = __float2bfloat16_rn(y);
        else e.k[(size_t)m * 256 + dim] = __float2bfloat16_rn(y);
      }
    } else if (nvalid) {
      // v^T: 16 consecutive tokens of one feature row -> 32 contiguous bytes
      const int d = n - e.q_features - 256;
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = pack_bf16(v[2 * j] * rs[c0 + 2 * j], v[2 * j + 1] * rs[c0 + 2 * j + 1]);
      uint4* dst = reinterpret_cast<uint4*>(e.vt + (size_t)d * e.vt_ld + m0);
      dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
      dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  } else if (KIND == EPI_RESID) {
    float xo[16];
#pragma unroll
    for (int j = 0; j < 16; ++j)  // all loads before the read-modify-write stores
      xo[j] = (nvalid && m0 + j < e.M) ? __ldcg(e.x + (size_t)(m0 + j) * e.N + n) : 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int m = m0 + j;
      float sq = 0.f;
      if (nvalid && m < e.M) {
        const size_t o = (size_t)m * e.N + n;
        const float xn = xo[j] + v[j];
        e.x[o] = xn;
        e.xb[o] = __float2bfloat16_rn(xn);
        sq = xn * xn;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
      if ((threadIdx.x & 31) == 0) red_q[c0 + j] = sq;
    }
  }
}

// NORMAL: thread = token m (fixed), columns = features n0 + j (16-aligned).
template <int KIND>
__device__ __forceinline__ void epi_normal(const EpiArgs& e, int m, int n0, float (&v)[16], float rs,
                                           float& ssq_acc, __nv_bfloat16* vbuf = nullptr) {
  // the warp-cooperative paths (V^T transpose, staged residual) need every
  // lane, valid row or not
  if (m >= e.M && !(KIND == EPI_QKV && vbuf && n0 >= e.q_features + 256) && !(KIND == EPI_RESID && vbuf))
    return;
  const bool full = n0 + 16 <= e.N;
  if (KIND == EPI_F32 || KIND == EPI_BF16 || KIND == EPI_TANH_BF16) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float o = v[j] * rs;
      if (e.bias && n0 + j < e.N) o += e.bias[n0 + j];
      if (KIND == EPI_TANH_BF16) o = tanh_fast(o);
      v[j] = o;
    }
    if (KIND == EPI_F32) {
      float* dst = e.out_f32 + (size_t)m * e.ld_f32 + n0;
      if (full && (e.ld_f32 % 4) == 0) {
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
        for (int j = 0; j < 16; ++j)
          if (n0 + j < e.N) dst[j] = v[j];
      }
    } else {
      __nv_bfloat16* dst = e.out_bf16 + (size_t)m * e.ld_bf16 + n0;
      if (full && (e.ld_bf16 % 8) == 0) {
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
      } else {
        for (int j = 0; j < 16; ++j)
          if (n0 + j < e.N) dst[j] = __float2bfloat16_rn(v[j]);
      }
    }
  } else if (KIND == EPI_GEGLU) {
    uint32_t w[4];
#pragma unroll
    for (int p = 0; p < 8; p += 2) {
      const float h0 = gelu_tanh(v[2 * p] * rs) * (v[2 * p + 1] * rs);
      const float h1 = gelu_tanh(v[2 * p + 2] * rs) * (v[2 * p + 3] * rs);
      w[p >> 1] = pack_bf16(h0, h1);
    }
    // 8 outputs h[n0/2 .. n0/2 + 7]
    *reinterpret_cast<uint4*>(e.out_bf16 + (size_t)m * e.ld_bf16 + (n0 >> 1)) =
        make_uint4(w[0], w[1], w[2], w[3]);
  } else if (KIND == EPI_QKV) {
    if (n0 < e.q_features + 256) {
      const int pos = e.pos0 + ((m % e.env_rows) % e.seg_len);
      const int i0 = (n0 & 255) >> 1;
      uint32_t wa[4], wb[4];
#pragma unroll
      for (int p = 0; p < 8; p += 2) {
        float ya[2], yb[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float a = v[2 * (p + u)] * rs, b = v[2 * (p + u) + 1] * rs;
          // table is position-fastest: a warp's consecutive tokens read consecutive entries
          const float2 cs = __ldg(e.rope + (size_t)(i0 + p + u) * e.rope_ld + pos);
          ya[u] = a * cs.x - b * cs.y;
          yb[u] = b * cs.x + a * cs.y;
        }
        wa[p >> 1] = pack_bf16(ya[0], ya[1]);
        wb[p >> 1] = pack_bf16(yb[0], yb[1]);
      }
      __nv_bfloat16* base = n0 < e.q_features ? e.q + (size_t)m * e.q_features + (n0 & ~255)
                                              : e.k + (size_t)m * 256;
      *reinterpret_cast<uint4*>(base + i0) = make_uint4(wa[0], wa[1], wa[2], wa[3]);
      *reinterpret_cast<uint4*>(base + 128 + i0) = make_uint4(wb[0], wb[1], wb[2], wb[3]);
    } else {
      const int d0 = n0 - e.q_features - 256;
      if (vbuf) {
        // V^T through a per-warp SMEM transpose: 16 features x 32 tokens, then
        // each lane stores two 16 B runs (8 consecutive tokens of one feature)
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int j = 0; j < 16; ++j) vbuf[j * 32 + lane] = __float2bfloat16_rn(v[j] * rs);
        __syncwarp();
        const int m0w = m - lane;  // first token of the warp
        const int d = lane >> 1;
        const int t0 = (lane & 1) * 16;  // 16 consecutive tokens of feature d: one 32 B store
        __nv_bfloat16* dst = e.vt + (size_t)(d0 + d) * e.vt_ld + m0w + t0;
        if (m0w + t0 + 15 < e.M && (e.vt_ld % 16) == 0) {
          const uint4 v0 = *reinterpret_cast<const uint4*>(vbuf + d * 32 + t0);
          const uint4 v1 = *reinterpret_cast<const uint4*>(vbuf + d * 32 + t0 + 8);
          const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
          st_global_v8(dst, w);
        } else {
          for (int z = 0; z < 16; ++z)
            if (m0w + t0 + z < e.M) dst[z] = vbuf[d * 32 + t0 + z];
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) e.vt[(size_t)(d0 + j) * e.vt_ld + m] = __float2bfloat16_rn(v[j] * rs);
      }
    }
  } else if (KIND == EPI_RESID) {
    if (vbuf) {
      // Coalesced residual update: the warp's 32 rows x 16 columns go through
      // a per-warp SMEM scratch so that every lane moves 32 contiguous bytes of
      // one row per instruction (LDG/STG.256 for x, 16 B for xb): 16 rows x
      // 64 B per x instruction, 16 rows x 32 B per xb instruction.
      float* sc = reinterpret_cast<float*>(vbuf);  // [32][16], quads XOR-swizzled by row
      const int lane = threadIdx.x & 31;
      const int m0w = m - lane;
#pragma unroll
      for (int qd = 0; qd < 4; ++qd)
        reinterpret_cast<float4*>(sc + lane * 16)[qd ^ (lane & 3)] =
            make_float4(v[4 * qd], v[4 * qd + 1], v[4 * qd + 2], v[4 * qd + 3]);
      __syncwarp();
      float rowsq[2];
      float xo[2][8];
      const int hq = lane & 1;  // columns [8 hq, 8 hq + 8) of the chunk
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {  // every residual load in flight first
        const int row = m0w + pass * 16 + (lane >> 1);
        if (row < e.M) {
          asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=f"(xo[pass][0]), "=f"(xo[pass][1]), "=f"(xo[pass][2]), "=f"(xo[pass][3]),
                         "=f"(xo[pass][4]), "=f"(xo[pass][5]), "=f"(xo[pass][6]), "=f"(xo[pass][7])
                       : "l"(e.x + (size_t)row * e.N + n0 + hq * 8));
        } else {
#pragma unroll
          for (int z = 0; z < 8; ++z) xo[pass][z] = 0.f;
        }
      }
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const int rr = pass * 16 + (lane >> 1);
        const int row = m0w + rr;
        const float4 a0 = reinterpret_cast<const float4*>(sc + rr * 16)[(2 * hq) ^ (rr & 3)];
        const float4 a1 = reinterpret_cast<const float4*>(sc + rr * 16)[(2 * hq + 1) ^ (rr & 3)];
        float y[8] = {xo[pass][0] + a0.x, xo[pass][1] + a0.y, xo[pass][2] + a0.z, xo[pass][3] + a0.w,
                      xo[pass][4] + a1.x, xo[pass][5] + a1.y, xo[pass][6] + a1.z, xo[pass][7] + a1.w};
        float sq = 0.f;
        if (row < e.M) {
          const uint32_t w[8] = {__float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]),
                                 __float_as_uint(y[3]), __float_as_uint(y[4]), __float_as_uint(y[5]),
                                 __float_as_uint(y[6]), __float_as_uint(y[7])};
          st_global_v8(e.x + (size_t)row * e.N + n0 + hq * 8, w);
          *reinterpret_cast<uint4*>(e.xb + (size_t)row * e.N + n0 + hq * 8) =
              make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]), pack_bf16(y[4], y[5]), pack_bf16(y[6], y[7]));
#pragma unroll
          for (int z = 0; z < 8; ++z) sq += y[z] * y[z];
        }
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        rowsq[pass] = sq;
      }
      // row rr's chunk sum back to its owner lane rr (lane (rr % 16) * 2 of pass rr / 16)
      float mine = 0.f;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const float t = __shfl_sync(0xffffffffu, rowsq[pass], (lane & 15) * 2);
        if ((lane >> 4) == pass) mine = t;
      }
      ssq_acc += mine;
      __syncwarp();
      return;
    }
    float* xr = e.x + (size_t)m * e.N + n0;
    __nv_bfloat16* xbr = e.xb + (size_t)m * e.N + n0;
    uint32_t w[8];
    float4 xin[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) xin[j] = reinterpret_cast<const float4*>(xr)[j];
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      float4 x4 = xin[j / 4];
      x4.x += v[j];
      x4.y += v[j + 1];
      x4.z += v[j + 2];
      x4.w += v[j + 3];
      *reinterpret_cast<float4*>(xr + j) = x4;
      ssq_acc += x4.x * x4.x + x4.y * x4.y + x4.z * x4.z + x4.w * x4.w;
      w[j / 2] = pack_bf16(x4.x, x4.y);
      w[j / 2 + 1] = pack_bf16(x4.z, x4.w);
    }
    reinterpret_cast<uint4*>(xbr)[0] = make_uint4(w[0], w[1], w[2], w[3]);
    reinterpret_cast<uint4*>(xbr)[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

// ------------------------------------------------------ shared mainloop parts

struct Ring {
  uint8_t* smem;
  uint64_t* full;
  uint64_t* empty;
  uint32_t stage_bytes, b_bytes;
  int stages;
};

// Producer for one tile's K range; `kiter` continues the ring across tiles.
__device__ __forceinline__ void produce_tile(const Ring& r, const CUtensorMap* tw,
                                             const CUtensorMap* tx, uint32_t w_off, uint32_t x_off,
                                             int w_row, int x_row, int kb0, int nkb, int& kiter,
                                             bool first_tile, uint64_t pol_w, uint64_t pol_x) {
  int i = 0;
  if (first_tile) {
    // weights first (independent of the previous kernel), then the PDL wait
    const int pre = min(r.stages, nkb);
    for (; i < pre; ++i) {
      const int s = (kiter + i) % r.stages;
      uint8_t* st = r.smem + s * r.stage_bytes;
      sm100::mbar_arrive_expect_tx(&r.full[s], kAStageBytes + r.b_bytes);
      sm100::tma_load_2d(tw, &r.full[s], st + w_off, (kb0 + i) * BK, w_row, pol_w);
    }
    sm100::pdl_wait();
    for (int u = 0; u < pre; ++u) {
      const int s = (kiter + u) % r.stages;
      sm100::tma_load_2d(tx, &r.full[s], r.smem + s * r.stage_bytes + x_off, (kb0 + u) * BK, x_row,
                         pol_x);
    }
  }
  for (; i < nkb; ++i) {
    const int k = kiter + i;
    const int s = k % r.stages;
    if (k >= r.stages) sm100::mbar_wait(&r.empty[s], ((k / r.stages) & 1) ^ 1);
    uint8_t* st = r.smem + s * r.stage_bytes;
    sm100::mbar_arrive_expect_tx(&r.full[s], kAStageBytes + r.b_bytes);
    sm100::tma_load_2d(tw, &r.full[s], st + w_off, (kb0 + i) * BK, w_row, pol_w);
    sm100::tma_load_2d(tx, &r.full[s], st + x_off, (kb0 + i) * BK, x_row, pol_x);
  }
  kiter += nkb;
}

__device__ __forceinline__ void mma_tile(const Ring& r, uint32_t tmem_d, uint32_t idesc, int nkb,
                                         int& kiter) {
  for (int i = 0; i < nkb; ++i) {
    const int k = kiter + i;
    const int s = k % r.stages;
    sm100::mbar_wait(&r.full[s], (k / r.stages) & 1);
    sm100::tc_fence_after();
    const uint32_t a_addr = sm100::smem_u32(r.smem + s * r.stage_bytes);
    const uint32_t b_addr = a_addr + kAStageBytes;
#pragma unroll
    for (int kk = 0; kk < BK / 16; ++kk)
      sm100::umma_bf16(tmem_d, sm100::make_sw128_desc(a_addr + kk * 32),
                       sm100::make_sw128_desc(b_addr + kk * 32), idesc, (i | kk) != 0);
    sm100::umma_commit(&r.empty[s]);
  }
  kiter += nkb;
}

// smem tail layout after the ring region
struct Tail {
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tmem_full;   // [2]
  uint64_t* tmem_empty;  // [2]
  uint32_t* tmem_slot;
  float* rs;             // [256]
  float* red;            // [4][256]
  float* sred;           // [2][2][128] (normal-mode ssq partials per warp group)
  __nv_bfloat16* vbuf;   // [8 warps][2 KB] epilogue staging (V^T transpose, residual)
};

__device__ __forceinline__ Tail carve_tail(uint8_t* smem, const Params& p) {
  Tail t;
  uint8_t* q = smem + p.smem_stage_region;
  t.full = reinterpret_cast<uint64_t*>(q);
  t.empty = t.full + p.stages;
  t.tmem_full = t.empty + p.stages;
  t.tmem_empty = t.tmem_full + 2;
  t.tmem_slot = reinterpret_cast<uint32_t*>(t.tmem_empty + 2);
  t.rs = reinterpret_cast<float*>(t.tmem_slot + 4);
  t.red = t.rs + 256;
  t.sred = t.red + 4 * 256;
  t.vbuf = reinterpret_cast<__nv_bfloat16*>(t.sred + 2 * 2 * 128);
  return t;
}

constexpr size_t kTailBytes = 8 * (2 * 16 + 4) + 16 + 4 * (256 + 4 * 256 + 2 * 2 * 128) + 8 * 2048;

// -------------------------------------------------- batch-1: swap + cluster split-K

__device__ __forceinline__ void stamp(const Params& p, int i) {
  if (p.dbg && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.dbg[i] = t;
  }
}

// Split-K finish for the chunks cluster rank `split` owns (ch % S == split,
// alternating between the two column groups g): G chunks at a time with up to
// 4 split partials per chunk in flight (16 float4 loads per thread),
// summed in fixed split order so the result is deterministic.
template <int KIND, int G>
__device__ __forceinline__ void reduce_chunks(const EpiArgs& e, const Params& p, const float* base,
                                              size_t sstride, int split, int g, int n, int tile_b,
                                              int nchunks, const float* rs, float* red) {
  constexpr int SB = 4 / G;  // splits per load batch
  const int S = p.splits;
  // owned chunks: split + k * S for k = g, g + 2, ...
  const int owned = (nchunks - split + S - 1) / S;
  const int cnt = (owned - g + 1) / 2;
#define mine(i) (split + (g + 2 * (i)) * S)
  for (int i0 = 0; i0 < cnt; i0 += G) {
    float v[G][16];
#pragma unroll
    for (int c = 0; c < G; ++c)
#pragma unroll
      for (int j = 0; j < 16; ++j) v[c][j] = 0.f;
    for (int s0 = 0; s0 < S; s0 += SB) {
      float4 a[G][SB][4];
#pragma unroll
      for (int c = 0; c < G; ++c)
#pragma unroll
        for (int u = 0; u < SB; ++u)
          if (i0 + c < cnt && s0 + u < S) {
            const float4* ps = reinterpret_cast<const float4*>(base + (size_t)(s0 + u) * sstride +
                                                               (size_t)mine(i0 + c) * BM * 16);
#pragma unroll
            for (int j = 0; j < 4; ++j) a[c][u][j] = __ldcg(ps + j * BM);
          }
#pragma unroll
      for (int c = 0; c < G; ++c)
#pragma unroll
        for (int u = 0; u < SB; ++u)
          if (i0 + c < cnt && s0 + u < S) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              v[c][4 * j] += a[c][u][j].x;
              v[c][4 * j + 1] += a[c][u][j].y;
              v[c][4 * j + 2] += a[c][u][j].z;
              v[c][4 * j + 3] += a[c][u][j].w;
            }
          }
    }
#pragma unroll
    for (int c = 0; c < G; ++c)
      if (i0 + c < cnt) epi_swap<KIND>(e, n, tile_b * p.bn + mine(i0 + c) * 16, v[c], rs, red, mine(i0 + c) * 16);
  }
#undef mine
}

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_swap_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                     const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Tail T = carve_tail(smem, p);
  const uint32_t b_bytes = (uint32_t)p.bn * BK * 2;
  const Ring ring{smem, T.full, T.empty, kAStageBytes + ((b_bytes + 1023) & ~1023u), b_bytes, p.stages};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_a = blockIdx.x, tile_b = blockIdx.y, split = blockIdx.z;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kb_per_split, p.num_kb - kb0);
  const int S = p.splits;
  if (threadIdx.x == 0) stamp(p, 0);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      sm100::mbar_init(&T.full[s], 1);
      sm100::mbar_init(&T.empty[s], 1);
    }
    sm100::mbar_init(&T.tmem_full[0], 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<256>(T.tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *T.tmem_slot;
  if (threadIdx.x == 0) stamp(p, 1);

  if (warp == 0) {
    if (sm100::elect_one()) {
      sm100::tma_prefetch_desc(&tma_a);
      sm100::tma_prefetch_desc(&tma_b);
      int kiter = 0;
      produce_tile(ring, &tma_a, &tma_b, 0, kAStageBytes, tile_a * BM, tile_b * p.bn, kb0, nkb,
                   kiter, true, sm100::policy_evict_first(), sm100::policy_evict_last());
      stamp(p, 2);
    }
  } else if (warp == 1) {
    if (sm100::elect_one()) {
      int kiter = 0;
      mma_tile(ring, tmem, sm100::make_idesc_bf16(BM, p.bn), nkb, kiter);
      sm100::umma_commit(&T.tmem_full[0]);
      stamp(p, 3);
    }
    __syncwarp();
  }

  // ---------------------------------------------------------------- epilogue
  const bool epi = warp >= 2;
  const int q = warp & 3;                 // TMEM lane quarter
  const int g = epi ? (warp - 2) >> 2 : 0;  // column group (0/1)
  const int lane_row = q * 32 + lane;
  const int n = tile_a * BM + lane_row;   // feature of this thread
  const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
  const EpiArgs& e = p.e;
  if (epi) {
    sm100::pdl_wait();
    if (threadIdx.x == 64) sm100::pdl_launch_dependents();
    for (int c = threadIdx.x - 64; c < p.bn; c += kEpiThreads) {
      const int m = tile_b * p.bn + c;
      T.rs[c] = (KIND != EPI_RESID && KIND != EPI_TANH_BF16 && m < e.M) ? row_scale(e, m) : 1.f;
    }
    if (threadIdx.x == 64) stamp(p, 4);
    sm100::mbar_wait(&T.tmem_full[0], 0);
    sm100::tc_fence_after();
    if (threadIdx.x == 64) stamp(p, 5);
  }
  const int nchunks = p.bn / 16;
  if (S == 1) {
    if (epi) {
      epi_bar();
      for (int ch = g; ch < nchunks; ch += 4) {  // two TMEM loads in flight per wait
        const bool two = ch + 2 < nchunks;
        uint32_t r[2][16];
        sm100::tmem_ld16(t_lane + ch * 16, r[0]);
        if (two) sm100::tmem_ld16(t_lane + (ch + 2) * 16, r[1]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !two) break;
          const int c = ch + 2 * u;
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[u][j]);
          epi_swap<KIND>(e, n, tile_b * p.bn + c * 16, v, T.rs, T.red + q * 256, c * 16);
        }
      }
      if (KIND == EPI_RESID) {
        epi_bar();
        for (int c = threadIdx.x - 64; c < p.bn; c += kEpiThreads) {
          const int m = tile_b * p.bn + c;
          if (m < e.M)
            e.ssq_out[(size_t)tile_a * e.ssq_out_ld + m] =
                ((T.red[c] + T.red[256 + c]) + T.red[512 + c]) + T.red[768 + c];
        }
      }
    }
  } else {
    // Split-K reduction through L2: every split writes its partial as
    // [chunk][4 col quads][128 lanes][4 cols] (each warp store is 512
    // contiguous bytes), one
    // cluster barrier, then chunk ch is reduced (fixed split order, so the
    // result is deterministic) and finished by cluster rank ch % S, reading
    // the S partials with 16-byte L2 loads. All S CTAs reduce in parallel.
    const int tile_id = tile_a * p.tiles_b + tile_b;
    const size_t slab = (size_t)nchunks * BM * 16;  // floats per (split, tile)
    float* mine = p.ws + ((size_t)split * p.total_tiles + tile_id) * slab;
    if (epi) {
      for (int ch = g; ch < nchunks; ch += 8) {  // four TMEM loads in flight per wait
        uint32_t r[4][16];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (ch + 2 * u < nchunks) sm100::tmem_ld16(t_lane + (ch + 2 * u) * 16, r[u]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (ch + 2 * u >= nchunks) break;
          float4* dst = reinterpret_cast<float4*>(mine + (size_t)(ch + 2 * u) * BM * 16) + lane_row;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[j * BM] = make_float4(__uint_as_float(r[u][4 * j]), __uint_as_float(r[u][4 * j + 1]),
                                      __uint_as_float(r[u][4 * j + 2]), __uint_as_float(r[u][4 * j + 3]));
        }
      }
    }
    if (threadIdx.x == 64) stamp(p, 6);
    // barrier.cluster arrive.release / wait.acquire orders the partial stores
    // before the peers' loads (cluster scope covers global memory)
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();  // every split's partial is in L2
    if (threadIdx.x == 64) stamp(p, 7);
    if (epi) {
      const float* base = p.ws + (size_t)tile_id * slab + lane_row * 4;
      const size_t sstride = (size_t)p.total_tiles * slab;
      if (S <= 2)
        reduce_chunks<KIND, 2>(e, p, base, sstride, split, g, n, tile_b, nchunks, T.rs, T.red + q * 256);
      else
        reduce_chunks<KIND, 1>(e, p, base, sstride, split, g, n, tile_b, nchunks, T.rs, T.red + q * 256);
    }
    if (threadIdx.x == 64) stamp(p, 8);
    if (KIND == EPI_RESID && epi) {
      epi_bar();
      for (int c = threadIdx.x - 64; c < p.bn; c += kEpiThreads) {
        const int m = tile_b * p.bn + c;
        if ((c >> 4) % S == split && m < e.M)
          e.ssq_out[(size_t)tile_a * e.ssq_out_ld + m] =
              ((T.red[c] + T.red[256 + c]) + T.red[512 + c]) + T.red[768 + c];
      }
    }
  }
  if (threadIdx.x == 64) stamp(p, 10);
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<256>(tmem);
  }
  if (threadIdx.x == 32) stamp(p, 11);
}

// ------------------------------------------------------ batched: persistent

// tiles a batched kernel visits: all, or the row tiles holding the live rows
// (*rows_dev * rows_mul, written before this kernel by the replanning graph)
__device__ __forceinline__ int live_tiles(const Params& p, int tile_rows, int tiles_b) {
  if (!p.rows_dev) return p.total_tiles;
  int r = __ldg(p.rows_dev) * p.rows_mul;
  r = r < p.rows_a ? r : p.rows_a;
  return ((r + tile_rows - 1) / tile_rows) * tiles_b;
}

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_persistent_kernel(const __grid_constant__ CUtensorMap tma_a,
                           const __grid_constant__ CUtensorMap tma_b, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Tail T = carve_tail(smem, p);
  const uint32_t b_bytes = (uint32_t)p.bn * BK * 2;
  const Ring ring{smem, T.full, T.empty, kAStageBytes + ((b_bytes + 1023) & ~1023u), b_bytes, p.stages};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      sm100::mbar_init(&T.full[s], 1);
      sm100::mbar_init(&T.empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&T.tmem_full[a], 1);
      sm100::mbar_init(&T.tmem_empty[a], kEpiThreads);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<512>(T.tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *T.tmem_slot;
  const int live = live_tiles(p, BM, p.tiles_b);

  if (warp == 0) {
    if (sm100::elect_one()) {
      sm100::tma_prefetch_desc(&tma_a);
      sm100::tma_prefetch_desc(&tma_b);
      const uint64_t pol_w = sm100::policy_evict_last();   // weights: reused by every row tile
      const uint64_t pol_x = sm100::policy_evict_first();  // activations: read by tiles_b CTAs at once
      int kiter = 0;
      bool first = true;
      for (int t = blockIdx.x; t < live; t += gridDim.x) {
        const int ta = t / p.tiles_b, tb = t % p.tiles_b;
        produce_tile(ring, &tma_b, &tma_a, kAStageBytes, 0, tb * p.bn, ta * BM, 0, p.num_kb, kiter,
                     first, pol_w, pol_x);
        first = false;
      }
    }
  } else if (warp == 1) {
    if (sm100::elect_one()) {
      const uint32_t idesc = sm100::make_idesc_bf16(BM, p.bn);
      int kiter = 0, it = 0;
      for (int t = blockIdx.x; t < live; t += gridDim.x, ++it) {
        const int a = it & 1;
        if (it >= 2) sm100::mbar_wait(&T.tmem_empty[a], ((it >> 1) & 1) ^ 1);
        sm100::tc_fence_after();
        mma_tile(ring, tmem + a * 256, idesc, p.num_kb, kiter);
        sm100::umma_commit(&T.tmem_full[a]);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int g = (warp - 2) >> 2;
    const int lane_row = q * 32 + lane;
    const EpiArgs& e = p.e;
    sm100::pdl_wait();
    if (threadIdx.x == 64) sm100::pdl_launch_dependents();
    int it = 0;
    for (int t = blockIdx.x; t < live; t += gridDim.x, ++it) {
      const int ta = t / p.tiles_b, tb = t % p.tiles_b;
      const int a = it & 1;
      const int m = ta * BM + lane_row;
      const float rs = (KIND != EPI_RESID && KIND != EPI_TANH_BF16 && m < e.M) ? row_scale(e, m) : 1.f;
      sm100::mbar_wait(&T.tmem_full[a], (it >> 1) & 1);
      sm100::tc_fence_after();
      const uint32_t t_lane = tmem + a * 256 + ((uint32_t)(q * 32) << 16);
      float ssq0 = 0.f, ssq1 = 0.f;
      const int nch = p.bn / 16;
      for (int ch = g; ch < nch; ch += 4) {  // two TMEM loads in flight per wait
        const bool two = ch + 2 < nch;
        uint32_t r[2][16];
        sm100::tmem_ld16(t_lane + ch * 16, r[0]);
        if (two) sm100::tmem_ld16(t_lane + (ch + 2) * 16, r[1]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !two) break;
          const int c = ch + 2 * u;
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[u][j]);
          float acc = 0.f;
          epi_normal<KIND>(e, m, tb * p.bn + c * 16, v, rs, acc, T.vbuf + (warp - 2) * 1024);
          if (c * 16 < 128) ssq0 += acc;
          else ssq1 += acc;
        }
      }
      float ssq[2] = {ssq0, ssq1};
      sm100::tc_fence_before();
      sm100::mbar_arrive(&T.tmem_empty[a]);
      if (KIND == EPI_RESID) {
        // two warp groups hold partial sums of the same 128-feature group
        T.sred[(g * 2 + 0) * 128 + lane_row] = ssq[0];
        T.sred[(g * 2 + 1) * 128 + lane_row] = ssq[1];
        epi_bar();
        if (g == 0 && m < e.M) {
          for (int fg = 0; fg < p.bn / 128; ++fg)
            e.ssq_out[(size_t)((tb * p.bn) / 128 + fg) * e.ssq_out_ld + m] =
                T.sred[fg * 128 + lane_row] + T.sred[(2 + fg) * 128 + lane_row];
        }
        epi_bar();
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------- batched: 2-SM CTA pairs
//
// gemm_pair_kernel: the batched GEMM on CTA pairs (cluster of 2 on one TPC)
// with tcgen05.mma.cta_group::2: one 256 x 256 tile per pair and k-block,
// CTA rank r holds A rows [r*128, r*128+128) and B rows (features)
// [r*128, r*128+128) of the tile; the pair's MMA reads both halves, so each
// SM loads 32 KB per 64-deep k-block instead of 48 KB for a 128 x 256 tile
// (the L2 -> SMEM ingress, ~93 GB/s per SM measured, is what bounds the
// 1-SM kernel). Only the leader (rank 0) issues MMAs; its full barrier counts
// the bytes of both CTAs' TMA loads (the peer signals it through
// .cta_group::2), the commit is multicast to both CTAs' empty / tmem_full
// barriers, and both CTAs' epilogue threads release the leader's tmem_empty.
// Each CTA's TMEM holds its own 128 rows x 256 columns (two accumulators).

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// TMA load whose completion is counted on the leader CTA's mbarrier.
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* m, uint32_t bar_cluster, void* dst,
                                                 int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(sm100::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          sm100::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// Release of a TMEM accumulator to the leader: only the epilogue's tcgen05.ld
// (waited, then tcgen05.fence::before_thread_sync) must precede it, not its
// global stores, so the arrive is relaxed (a .release.cluster arrive makes
// every thread wait for its stores: MEMBAR + ERRBAR, 10 % of the QKV
// kernel's stall samples) and issued once per warp.
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
               : "memory");
}

constexpr uint32_t kPairStageBytes = 2 * BM * BK * 2;  // A half + B half: 32 KB

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tma_a,
                     const __grid_constant__ CUtensorMap tma_b, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Tail T = carve_tail(smem, p);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int tiles_n = p.tiles_b;  // 256-feature tiles
  cg::cluster_group cluster = cg::this_cluster();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      sm100::mbar_init(&T.full[s], 1);
      sm100::mbar_init(&T.empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&T.tmem_full[a], 1);
      sm100::mbar_init(&T.tmem_empty[a], 2 * kEpiWarps);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        sm100::smem_u32(T.tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  sm100::tc_fence_before();
  cluster.sync();  // barriers of both CTAs initialised, TMEM allocated in both
  sm100::tc_fence_after();
  const uint32_t tmem = *T.tmem_slot;
  const int live = live_tiles(p, 256, tiles_n);

  if (warp == 0) {
    if (sm100::elect_one()) {
      sm100::tma_prefetch_desc(&tma_a);
      sm100::tma_prefetch_desc(&tma_b);
      const uint64_t pol_w = sm100::policy_evict_last();
      // activations too: the tiles_n pairs sharing an A row block run at about
      // the same time, and evict_first let lagging readers miss to HBM
      // (QKV read 4x its A bytes from DRAM); evict_last: -3 % on the batched
      // GEMMs (evict_normal: -1.5 %)
      const uint64_t pol_x = sm100::policy_evict_last();
      int kiter = 0;
      bool first = true;
      for (int t = pair; t < live; t += n_pairs) {
        const int tm = t / tiles_n, tn = t % tiles_n;
        const int a_row = tm * 256 + rank * BM, b_row = tn * 256 + rank * BM;
        for (int i = 0; i < p.num_kb; ++i, ++kiter) {
          const int s = kiter % p.stages;
          if (kiter >= p.stages) sm100::mbar_wait(&T.empty[s], ((kiter / p.stages) & 1) ^ 1);
          uint8_t* st = smem + (size_t)s * kPairStageBytes;
          const uint32_t fb = mapa_shared(sm100::smem_u32(&T.full[s]), 0);
          if (leader) sm100::mbar_arrive_expect_tx(&T.full[s], 2 * kPairStageBytes);
          tma_load_2d_pair(&tma_b, fb, st + BM * BK * 2, i * BK, b_row, pol_w);
          if (first && i == 0) sm100::pdl_wait();  // weights before, activations after
          tma_load_2d_pair(&tma_a, fb, st, i * BK, a_row, pol_x);
        }
        first = false;
      }
    }
  } else if (warp == 1) {
    if (leader && sm100::elect_one()) {
      const uint32_t idesc = sm100::make_idesc_bf16(256, 256);
      int kiter = 0, it = 0;
      for (int t = pair; t < live; t += n_pairs, ++it) {
        const int a = it & 1;
        if (it >= 2) sm100::mbar_wait(&T.tmem_empty[a], ((it >> 1) & 1) ^ 1);
        sm100::tc_fence_after();
        for (int i = 0; i < p.num_kb; ++i, ++kiter) {
          const int s = kiter % p.stages;
          sm100::mbar_wait(&T.full[s], (kiter / p.stages) & 1);
          sm100::tc_fence_after();
          const uint32_t a_addr = sm100::smem_u32(smem + (size_t)s * kPairStageBytes);
          const uint32_t b_addr = a_addr + BM * BK * 2;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16_pair(tmem + a * 256, sm100::make_sw128_desc(a_addr + kk * 32),
                           sm100::make_sw128_desc(b_addr + kk * 32), idesc, (i | kk) != 0);
          umma_commit_pair(&T.empty[s]);
        }
        umma_commit_pair(&T.tmem_full[a]);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int g = (warp - 2) >> 2;
    const int lane_row = q * 32 + lane;
    const EpiArgs& e = p.e;
    const uint32_t te = mapa_shared(sm100::smem_u32(&T.tmem_empty[0]), 0);
    sm100::pdl_wait();
    if (threadIdx.x == 64) sm100::pdl_launch_dependents();
    int it = 0;
    for (int t = pair; t < live; t += n_pairs, ++it) {
      const int tm = t / tiles_n, tn = t % tiles_n;
      const int a = it & 1;
      const int m = tm * 256 + rank * BM + lane_row;
      const float rs = (KIND != EPI_RESID && KIND != EPI_TANH_BF16 && m < e.M) ? row_scale(e, m) : 1.f;
      sm100::mbar_wait(&T.tmem_full[a], (it >> 1) & 1);
      sm100::tc_fence_after();
      const uint32_t t_lane = tmem + a * 256 + ((uint32_t)(q * 32) << 16);
      float ssq0 = 0.f, ssq1 = 0.f;
      if (KIND == EPI_QKV && tn * 256 < e.q_features + 256) {
        // q / k head tile with RoPE: adjacent chunks (c, c+1) per pass, so each
        // row's rotated halves leave as 32 B runs (dims [8c, 8c+16) and
        // [128+8c, 128+8c+16)) -- full L2 sectors instead of 16 B pieces
        const int pos = m < e.M ? e.pos0 + ((m % e.env_rows) % e.seg_len) : 0;
        __nv_bfloat16* base = tn * 256 < e.q_features ? e.q + (size_t)m * e.q_features + tn * 256
                                                      : e.k + (size_t)m * 256;
        for (int c = 2 * g; c < 16; c += 4) {
          uint32_t r[2][16];
          sm100::tmem_ld16(t_lane + c * 16, r[0]);
          sm100::tmem_ld16(t_lane + (c + 1) * 16, r[1]);
          sm100::tmem_ld_wait();
          uint32_t wa[8], wb[8];
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int pp = 0; pp < 8; pp += 2) {
              float ya[2], yb[2];
#pragma unroll
              for (int w2 = 0; w2 < 2; ++w2) {
                const int pr = pp + w2;  // pair index inside the chunk
                const float x0 = __uint_as_float(r[u][2 * pr]) * rs, x1 = __uint_as_float(r[u][2 * pr + 1]) * rs;
                const float2 cs = __ldg(e.rope + (size_t)((c + u) * 8 + pr) * e.rope_ld + pos);
                ya[w2] = x0 * cs.x - x1 * cs.y;
                yb[w2] = x1 * cs.x + x0 * cs.y;
              }
              wa[u * 4 + (pp >> 1)] = pack_bf16(ya[0], ya[1]);
              wb[u * 4 + (pp >> 1)] = pack_bf16(yb[0], yb[1]);
            }
          if (m < e.M) {
            st_global_v8(base + c * 8, wa);
            st_global_v8(base + 128 + c * 8, wb);
          }
        }
      } else if (KIND == EPI_RESID && tn * 256 + 256 <= e.N) {
        // residual chunks: the next pass's x rows are loaded before this pass's
        // TMEM loads are consumed (two chunk pairs of loads in flight)
        float* sc = reinterpret_cast<float*>(T.vbuf + (warp - 2) * 1024);  // [32][16] staging
        const int m0w = m - lane;
        float xo[2][2][8];
        resid_load(e.x, e.M, e.N, m0w, tn * 256 + g * 16, lane, xo[0]);
        resid_load(e.x, e.M, e.N, m0w, tn * 256 + (g + 2) * 16, lane, xo[1]);
        for (int ch = g; ch < 16; ch += 4) {
          uint32_t r[2][16];
          sm100::tmem_ld16(t_lane + ch * 16, r[0]);
          sm100::tmem_ld16(t_lane + (ch + 2) * 16, r[1]);
          sm100::tmem_ld_wait();
          float xn[2][2][8];
          if (ch + 4 < 16) {
            resid_load(e.x, e.M, e.N, m0w, tn * 256 + (ch + 4) * 16, lane, xn[0]);
            resid_load(e.x, e.M, e.N, m0w, tn * 256 + (ch + 6) * 16, lane, xn[1]);
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int n0 = tn * 256 + (ch + 2 * u) * 16;
#pragma unroll
            for (int qd = 0; qd < 4; ++qd)
              reinterpret_cast<float4*>(sc + lane * 16)[qd ^ (lane & 3)] =
                  make_float4(__uint_as_float(r[u][4 * qd]), __uint_as_float(r[u][4 * qd + 1]),
                              __uint_as_float(r[u][4 * qd + 2]), __uint_as_float(r[u][4 * qd + 3]));
            __syncwarp();
            const int hq = lane & 1;
            float rowsq[2];
#pragma unroll
            for (int pass = 0; pass < 2; ++pass) {
              const int rr = pass * 16 + (lane >> 1);
              const int row = m0w + rr;
              const float4 a0 = reinterpret_cast<const float4*>(sc + rr * 16)[(2 * hq) ^ (rr & 3)];
              const float4 a1 = reinterpret_cast<const float4*>(sc + rr * 16)[(2 * hq + 1) ^ (rr & 3)];
              const float* xv = xo[u][pass];
              const float y[8] = {xv[0] + a0.x, xv[1] + a0.y, xv[2] + a0.z, xv[3] + a0.w,
                                  xv[4] + a1.x, xv[5] + a1.y, xv[6] + a1.z, xv[7] + a1.w};
              float sq = 0.f;
              if (row < e.M) {
                const uint32_t w[8] = {__float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]),
                                       __float_as_uint(y[3]), __float_as_uint(y[4]), __float_as_uint(y[5]),
                                       __float_as_uint(y[6]), __float_as_uint(y[7])};
                st_global_v8(e.x + (size_t)row * e.N + n0 + hq * 8, w);
                *reinterpret_cast<uint4*>(e.xb + (size_t)row * e.N + n0 + hq * 8) =
                    make_uint4(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]), pack_bf16(y[4], y[5]),
                               pack_bf16(y[6], y[7]));
#pragma unroll
                for (int z = 0; z < 8; ++z) sq += y[z] * y[z];
              }
              sq += __shfl_xor_sync(0xffffffffu, sq, 1);
              rowsq[pass] = sq;
            }
            float mine = 0.f;
#pragma unroll
            for (int pass = 0; pass < 2; ++pass) {
              const float t2 = __shfl_sync(0xffffffffu, rowsq[pass], (lane & 15) * 2);
              if ((lane >> 4) == pass) mine = t2;
            }
            if ((ch + 2 * u) * 16 < 128) ssq0 += mine;
            else ssq1 += mine;
            __syncwarp();
          }
          if (ch + 4 < 16) {
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int pass = 0; pass < 2; ++pass)
#pragma unroll
                for (int z = 0; z < 8; ++z) xo[u][pass][z] = xn[u][pass][z];
          }
        }
      } else if (KIND == EPI_GEGLU && (e.ld_bf16 % 16) == 0 && tn * 256 + 256 <= e.N) {
        // adjacent chunk pairs: 16 consecutive outputs h[128 tn + 8c, +16) per
        // row leave as one 32 B store (full L2 sector)
        __nv_bfloat16* hrow = e.out_bf16 + (size_t)m * e.ld_bf16 + tn * 128;
        for (int c = 2 * g; c < 16; c += 4) {
          uint32_t r[2][16];
          sm100::tmem_ld16(t_lane + c * 16, r[0]);
          sm100::tmem_ld16(t_lane + (c + 1) * 16, r[1]);
          sm100::tmem_ld_wait();
          uint32_t w[8];
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int pp = 0; pp < 8; pp += 2) {
              const float h0 = gelu_tanh(__uint_as_float(r[u][2 * pp]) * rs) * (__uint_as_float(r[u][2 * pp + 1]) * rs);
              const float h1 =
                  gelu_tanh(__uint_as_float(r[u][2 * pp + 2]) * rs) * (__uint_as_float(r[u][2 * pp + 3]) * rs);
              w[u * 4 + (pp >> 1)] = pack_bf16(h0, h1);
            }
          if (m < e.M) st_global_v8(hrow + c * 8, w);
        }
      } else
      for (int ch = g; ch < 16; ch += 4) {  // two TMEM loads in flight per wait
        uint32_t r[2][16];
        sm100::tmem_ld16(t_lane + ch * 16, r[0]);
        sm100::tmem_ld16(t_lane + (ch + 2) * 16, r[1]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = ch + 2 * u;
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[u][j]);
          float acc = 0.f;
          if (tn * 256 + c * 16 < e.N)
            epi_normal<KIND>(e, m, tn * 256 + c * 16, v, rs, acc, T.vbuf + (warp - 2) * 1024);
          if (c * 16 < 128) ssq0 += acc;
          else ssq1 += acc;
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote_relaxed(te + a * 8);
      if (KIND == EPI_RESID) {
        T.sred[(g * 2 + 0) * 128 + lane_row] = ssq0;
        T.sred[(g * 2 + 1) * 128 + lane_row] = ssq1;
        epi_bar();
        if (g == 0 && m < e.M) {
          for (int fg = 0; fg < 2; ++fg)
            e.ssq_out[(size_t)(tn * 2 + fg) * e.ssq_out_ld + m] =
                T.sred[fg * 128 + lane_row] + T.sred[(2 + fg) * 128 + lane_row];
        }
        epi_bar();
      }
    }
  }
  sm100::tc_fence_before();
  cluster.sync();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    sm100::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace gemm
}  // namespace sf
