// fp32 mode of the pi0-scale Action Expert layer stack (sm_100a, CUDA cores).
//
// The north star's second precision mode ("1e-5 in an fp32 mode"): the same
// bf16 weights and prefix KV, every activation kept in fp32 and every dot
// product accumulated in fp32 FMA (SIMT; tcgen05 has no fp32-exact kind), so
// endpoints and distances match the unrounded fp32 model to fp32 rounding and
// prefix / fallback decisions can be compared at the 1e-4 band. It replaces
// only the layer stack + head (run_stack) of the verify / Euler chains; the
// embedding, verify epilogue and Euler update kernels are shared with the
// bf16 path. Not a performance path: ~10 ms per cfg3 verify.
//
// Per layer: rms -> QKV GEMM (x RMS row scale) -> RoPE / split -> MQA
// attention (exact softmax, masks as attention.cuh) -> O GEMM (+= residual) ->
// rms -> gate/up GEMM (x RMS) -> GeGLU -> down GEMM (+= residual); head:
// rms -> out GEMM (x RMS + bias). Device weight layouts as the bf16 path
// (q/k rows interleaved (i, i + 128), gate/up rows interleaved (gate_i, up_i)).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace sf {
namespace f32 {

// rs[m] = 1 / sqrt(mean_n x[m, n]^2 + eps): one warp per row
__global__ void rms_rows_kernel(const float* __restrict__ x, int M, int W, float eps,
                                float* __restrict__ rs) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= M) return;
  const float* r = x + (size_t)warp * W;
  float s = 0.f;
  for (int i = lane; i < W; i += 32) s = fmaf(r[i], r[i], s);
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) rs[warp] = 1.f / sqrtf(s / (float)W + eps);
}

enum Epi : int { E_STORE = 0, E_RESID = 1 };

// C[m, n] (op)= (sum_k A[m, k] * W[n, k]) * rs[m] + bias[n]
// A fp32 [M][K] (lda), W bf16 [N][K]; 64 x 64 tile per CTA, 256 threads x
// (4 x 4) outputs, 32-deep K chunks staged in SMEM (W converted to fp32).
// Accumulation runs sequentially over k per output (deterministic).
template <int EPI>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int lda,
                                                       const __nv_bfloat16* __restrict__ Wt,
                                                       int M, int N, int K, const float* __restrict__ rs,
                                                       const float* __restrict__ bias, float* C, int ldc) {
  constexpr int TM = 64, TN = 64, TK = 32;
  __shared__ float sa[TK][TM + 4];
  __shared__ float sw[TK][TN + 4];
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = threadIdx.x; i < TM * TK; i += 256) {
      const int r = i / TK, c = i - r * TK;
      const int m = m0 + r, k = k0 + c;
      sa[c][r] = (m < M && k < K) ? A[(size_t)m * lda + k] : 0.f;
      const int n = n0 + r;
      sw[c][r] = (n < N && k < K) ? __bfloat162float(Wt[(size_t)n * K + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < TK; ++c) {
      float a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sa[c][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = sw[c][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
    const float r = rs ? rs[m] : 1.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j] * r;
      if (bias) v += bias[n];
      float* dst = C + (size_t)m * ldc + n;
      if (EPI == E_RESID) *dst = *dst + v;
      else *dst = v;
    }
  }
}

struct RopeParams {
  const float* qkv;    // [M][(nh + 2) * 256] device row order
  const float2* rope;  // [128][rope_ld] (cos, sin), position fastest
  int rope_ld;
  int M, nh, env_rows, T, P;
  float* q;  // [M][nh][256] natural dims
  float* k;  // [M][256]
  float* v;  // [M][256]
};

// Device QKV rows (2i, 2i + 1) = natural dims (i, i + 128) of a head; RoPE
// rotate_half at position P + t (t = token index in its segment).
__global__ void rope_split_f32_kernel(const RopeParams p) {
  const int m = blockIdx.x;
  const int t = (m % p.env_rows) % p.T;
  const int pos = p.P + t;
  const int ld = (p.nh + 2) * 256;
  const float* row = p.qkv + (size_t)m * ld;
  for (int idx = threadIdx.x; idx < (p.nh + 1) * 128; idx += blockDim.x) {
    const int hh = idx >> 7, i = idx & 127;
    const float a = row[hh * 256 + 2 * i], b = row[hh * 256 + 2 * i + 1];
    const float2 cs = p.rope[(size_t)i * p.rope_ld + pos];
    const float lo = a * cs.x - b * cs.y, hi = b * cs.x + a * cs.y;
    float* dst = hh < p.nh ? p.q + ((size_t)m * p.nh + hh) * 256 : p.k + (size_t)m * 256;
    dst[i] = lo;
    dst[i + 128] = hi;
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) p.v[(size_t)m * 256 + i] = row[(p.nh + 1) * 256 + i];
}

struct AttnParams {
  const float* q;                // [M][nh][256]
  const float* k;                // [M][256] suffix keys
  const float* v;                // [M][256] suffix values
  const __nv_bfloat16* kp;       // layer's prefix K pool [E_pool][P][256]
  const __nv_bfloat16* vtp;      // layer's prefix V^T pool [E_pool][256][P]
  const int* env_map;            // [B] pool slot per batch env
  int M, B, nh, env_rows, T, K, P;
  float scale;
  float* o;  // [M][nh * 256]
};

// One CTA per token row, all heads (MQA: the heads share each key / value).
// Keys: the env's prefix, then its segment's suffix tokens (the state token
// sees only itself); exact softmax in fp32.
constexpr int NH = 8;  // query heads (sf_ae_create requires 8)
__global__ void __launch_bounds__(256) attn_f32_kernel(const AttnParams p) {
  extern __shared__ float sm[];
  float* sq = sm;                         // [NH][256]
  float* sp = sq + NH * 256;              // [NH][n_keys]
  __shared__ float stat[8][2];
  const int m = blockIdx.x;
  const int e = m / p.env_rows, local = m - e * p.env_rows;
  float* out = p.o + (size_t)m * p.nh * 256;
  if (e >= p.B || local >= p.K * p.T) {  // padding row
    for (int i = threadIdx.x; i < p.nh * 256; i += blockDim.x) out[i] = 0.f;
    return;
  }
  const int br = local / p.T, t = local - br * p.T;
  const int seg0 = e * p.env_rows + br * p.T;  // first suffix token of the segment
  const int n_suf = t == 0 ? 1 : p.T;
  const int n_keys = p.P + n_suf;
  const int slot = p.env_map ? p.env_map[e] : e;
  const __nv_bfloat16* kp = p.kp + (size_t)slot * p.P * 256;
  const __nv_bfloat16* vtp = p.vtp + (size_t)slot * 256 * p.P;
  for (int i = threadIdx.x; i < p.nh * 256; i += blockDim.x) sq[i] = p.q[(size_t)m * p.nh * 256 + i];
  __syncthreads();
  // scores: one thread per key, all heads (16-byte key loads)
  for (int j = threadIdx.x; j < n_keys; j += blockDim.x) {
    float s[8] = {};
    if (j < p.P) {
      const uint4* kr = reinterpret_cast<const uint4*>(kp + (size_t)j * 256);
      for (int d0 = 0; d0 < 32; ++d0) {
        const uint4 raw = kr[d0];
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2 kv = __bfloat1622float2(b2[u]);
          const int d = d0 * 8 + 2 * u;
          #pragma unroll
          for (int hh = 0; hh < NH; ++hh) {
            s[hh] = fmaf(sq[hh * 256 + d], kv.x, s[hh]);
            s[hh] = fmaf(sq[hh * 256 + d + 1], kv.y, s[hh]);
          }
        }
      }
    } else {
      const float4* kr = reinterpret_cast<const float4*>(p.k + (size_t)(seg0 + (t == 0 ? 0 : j - p.P)) * 256);
      for (int d0 = 0; d0 < 64; ++d0) {
        const float4 kv = kr[d0];
        const int d = d0 * 4;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
          s[hh] = fmaf(sq[hh * 256 + d], kv.x, s[hh]);
          s[hh] = fmaf(sq[hh * 256 + d + 1], kv.y, s[hh]);
          s[hh] = fmaf(sq[hh * 256 + d + 2], kv.z, s[hh]);
          s[hh] = fmaf(sq[hh * 256 + d + 3], kv.w, s[hh]);
        }
      }
    }
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) sp[hh * n_keys + j] = s[hh] * p.scale;
  }
  __syncthreads();
  // softmax per head: warp hh (of 8) reduces head hh
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < NH) {
    float* row = sp + warp * n_keys;
    float mx = -INFINITY;
    for (int j = lane; j < n_keys; j += 32) mx = fmaxf(mx, row[j]);
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    float sum = 0.f;
    for (int j = lane; j < n_keys; j += 32) {
      const float e_ = expf(row[j] - mx);
      row[j] = e_;
      sum += e_;
    }
    for (int off = 16; off; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (lane == 0) stat[warp][0] = sum;
  }
  __syncthreads();
  // PV: thread = output dim, all heads
  const int d = threadIdx.x;
  float acc[8] = {};
  const __nv_bfloat16* vr = vtp + (size_t)d * p.P;
  int j = 0;
  for (; j + 8 <= p.P; j += 8) {  // 8 keys per 16-byte load of the V^T row
    const uint4 raw = *reinterpret_cast<const uint4*>(vr + j);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float2 vv = __bfloat1622float2(b2[u]);
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        acc[hh] = fmaf(sp[hh * n_keys + j + 2 * u], vv.x, acc[hh]);
        acc[hh] = fmaf(sp[hh * n_keys + j + 2 * u + 1], vv.y, acc[hh]);
      }
    }
  }
  for (; j < p.P; ++j) {
    const float vv = __bfloat162float(vr[j]);
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) acc[hh] = fmaf(sp[hh * n_keys + j], vv, acc[hh]);
  }
  for (int j = 0; j < n_suf; ++j) {
    const float vv = p.v[(size_t)(seg0 + (t == 0 ? 0 : j)) * 256 + d];
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) acc[hh] = fmaf(sp[hh * n_keys + p.P + j], vv, acc[hh]);
  }
#pragma unroll
  for (int hh = 0; hh < NH; ++hh) out[hh * 256 + d] = acc[hh] / stat[hh][0];
}

// h[m, i] = gelu_tanh(gu[m, 2i]) * gu[m, 2i + 1] (rows interleaved gate/up)
__global__ void geglu_f32_kernel(const float* __restrict__ gu, int M, int F, float* __restrict__ h) {
  const size_t total = (size_t)M * F;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t m = i / F, j = i - m * F;
    const float g = gu[m * 2 * F + 2 * j], u = gu[m * 2 * F + 2 * j + 1];
    const float x3 = g * g * g;
    h[i] = 0.5f * g * (1.f + tanhf(0.7978845608028654f * (g + 0.044715f * x3))) * u;
  }
}

}  // namespace f32
}  // namespace sf
