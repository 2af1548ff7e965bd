// pi0-scale Action Expert: verify chain and Euler full path (sm_100a).
//
// Per verify round (B envs x K branches, T = 1 + H suffix tokens per branch,
// env_rows = K*T token rows per env, dense; rows padded to 16 at the end):
//   embed        x_t = tau a + (1-tau) eps (verifier.py:73) -> action_in + temb,
//                state_proj; fp32 residual X, bf16 copy, RMS partial sums
//   18 x layer   QKV GEMM (RMS scale + RoPE fused)  -> MQA attention vs the
//                shared prefix KV -> O GEMM (+residual) -> gate/up GEMM
//                (RMS scale + GeGLU fused) -> down GEMM (+residual)
//   head         out_proj GEMM (RMS scale + bias) -> velocity v
//   epilogue     recon = x + (1-tau) v, distances, warp-ballot prefix,
//                min over K, gripper gate, decision (verify_epi.cuh)
// The whole sequence is captured once per (B, K) shape into a CUDA graph with
// programmatic dependent launch between kernels; the Euler full path
// (flowpolicy.py:273-292) is N x (embed, layers, head, update) in one graph.

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdlib.h>

#include <map>
#include <tuple>
#include <memory>
#include <vector>

#include "attention.cuh"
#include "b1engine.cuh"
#include "common.cuh"
#include "gemm_host.h"
#include "gemm.cuh"
#include "stack_f32.cuh"
#include "replan.cuh"
#include "specflow_b200_internal.h"
#include "specflow_b200_pi0.h"
#include "verify_epi.cuh"

namespace sf {
namespace pi0 {

using bf16 = __nv_bfloat16;

// ----------------------------------------------------------- init kernel

__device__ __forceinline__ float hash_uniform(uint64_t seed, uint64_t tid, uint64_t idx, float a) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull + tid * 0xD1B54A32D192ED03ull + idx;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  const float u = __fmul_rn((float)(uint32_t)(z >> 40), 5.9604644775390625e-08f);  // 2^-24
  return __fmul_rn(__fsub_rn(__fmul_rn(u, 2.0f), 1.0f), a);
}

__global__ void fill_hash_kernel(void* dst, int is_bf16, int64_t n, uint64_t seed, uint64_t tid,
                                 float a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = hash_uniform(seed, tid, (uint64_t)i, a);
    if (is_bf16) static_cast<bf16*>(dst)[i] = __float2bfloat16_rn(v);
    else static_cast<float*>(dst)[i] = v;
  }
}

// --------------------------------------------------- time embedding (fp32)

// h = swish(W1 f(tau) + b1) for R taus; one warp per output feature.
__global__ void temb_hidden_kernel(const float* __restrict__ w1, const float* __restrict__ b1,
                                   const float* __restrict__ taus, int R, int W, float min_p,
                                   float max_p, float* __restrict__ hidden) {
  extern __shared__ float feat[];  // [R][W]
  const int half = W / 2;
  for (int idx = threadIdx.x; idx < R * W; idx += blockDim.x) {
    const int r = idx / W, i = idx - r * W;
    const int ii = i < half ? i : i - half;
    const double frac = half > 1 ? (double)ii / (double)(half - 1) : 0.0;
    const double period = (double)min_p * pow((double)max_p / (double)min_p, frac);
    const double ang = 2.0 * 3.141592653589793 * (double)taus[r] / period;
    feat[idx] = (float)(i < half ? sin(ang) : cos(ang));
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int o = blockIdx.x * nw + warp; o < W; o += gridDim.x * nw) {
    for (int r = 0; r < R; ++r) {
      float acc = 0.f;
      for (int i = lane; i < W; i += 32) acc = fmaf(w1[(size_t)o * W + i], feat[r * W + i], acc);
      for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) {
        const float h = acc + b1[o];
        hidden[r * W + o] = h / (1.f + expf(-h));
      }
    }
  }
}

__global__ void temb_out_kernel(const float* __restrict__ w2, const float* __restrict__ b2,
                                const float* __restrict__ hidden, int R, int W,
                                float* __restrict__ temb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int o = blockIdx.x * nw + warp; o < W; o += gridDim.x * nw) {
    for (int r = 0; r < R; ++r) {
      float acc = 0.f;
      for (int i = lane; i < W; i += 32) acc = fmaf(w2[(size_t)o * W + i], hidden[r * W + i], acc);
      for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) temb[r * W + o] = acc + b2[o];
    }
  }
}

// ------------------------------------------------------------ embedding

struct EmbedParams {
  int W, D, S, H, T, K, env_rows, B;
  int mode;             // 0: verify (interpolate draft/eps at taus[k]); 1: Euler (actions given)
  const float* draft;   // [B][H][D]   (mode 0) | current A [B][H][D] (mode 1)
  const float* eps;     // [B][H][D]   (mode 0)
  float taus[SF_MAX_K];
  const float* temb;    // [K][W] (mode 0) | [1][W] for this step (mode 1)
  const float* state;   // [B][S]
  const float* a_wt;    // [D][W] (transposed copy of a_w [W][D])
  const float* a_b;
  const float* s_wt;    // [S][W]
  const float* s_b;
  float* x;             // [M][W]
  bf16* xb;             // [M][W]
  float* ssq;           // [W/128][M_ld]
  int ssq_ld;
};

// One CTA per (16 token rows, 256 features): thread t owns feature
// blockIdx.y * 256 + t. The embedding weights are read through transposed
// copies ([D][W], [S][W], made once at sf_ae_create) so every weight load is
// a coalesced 1 KB warp access, and each is reused for all 16 tokens.
constexpr int kEmbedTok = 16;  // token rows per CTA (8 for batched rounds, see launch_embed)

template <int TOK>
__global__ void __launch_bounds__(256) embed_kernel(const EmbedParams p) {
  sm100::pdl_wait();
  const int m0 = blockIdx.x * TOK;
  __shared__ float in[TOK][65];
  __shared__ int kind[TOK];  // 0 padding, 1 state token, 2 action token
  __shared__ int kbr[TOK];   // branch of the token
  __shared__ float red[8][TOK];
  __shared__ int has_state;
  if (threadIdx.x == 0) has_state = 0;
  __syncthreads();
  for (int idx = threadIdx.x; idx < TOK * 64; idx += blockDim.x) {
    const int tk = idx >> 6, c = idx & 63;
    const int m = m0 + tk;
    const int e = m / p.env_rows;
    const int local = m - e * p.env_rows;
    const int k = local / p.T;
    const int t = local - k * p.T;
    const bool real = local < p.K * p.T && e < p.B;
    float v = 0.f;
    if (real) {
      if (t == 0) {
        if (c < p.S) v = p.state[e * p.S + c];
      } else if (c < p.D) {
        if (p.mode == 0) {
          const int i = (e * p.H + (t - 1)) * p.D + c;
          const float tau = p.taus[k];
          // tau * a + (1 - tau) * eps, rounded like the verify epilogue (verifier.py:73)
          v = __fadd_rn(__fmul_rn(tau, p.draft[i]), __fmul_rn(__fsub_rn(1.f, tau), p.eps[i]));
        } else {
          v = p.draft[((e * p.K + k) * p.H + (t - 1)) * p.D + c];
        }
      }
    }
    in[tk][c] = v;
    if (c == 0) {
      kind[tk] = real ? (t == 0 ? 1 : 2) : 0;
      kbr[tk] = k;
      if (real && t == 0) has_state = 1;
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = blockIdx.y * 256 + threadIdx.x;
  float acc[TOK];
  const float ab = p.a_b[n];
#pragma unroll
  for (int tk = 0; tk < TOK; ++tk) acc[tk] = ab;
#pragma unroll 8
  for (int c = 0; c < p.D; ++c) {
    const float w = __ldg(p.a_wt + c * p.W + n);
#pragma unroll
    for (int tk = 0; tk < TOK; ++tk) acc[tk] = fmaf(w, in[tk][c], acc[tk]);
  }
  if (has_state) {
    float sacc[TOK];
    const float sb = p.s_b[n];
#pragma unroll
    for (int tk = 0; tk < TOK; ++tk) sacc[tk] = sb;
#pragma unroll 8
    for (int c = 0; c < p.S; ++c) {
      const float w = __ldg(p.s_wt + c * p.W + n);
#pragma unroll
      for (int tk = 0; tk < TOK; ++tk) sacc[tk] = fmaf(w, in[tk][c], sacc[tk]);
    }
#pragma unroll
    for (int tk = 0; tk < TOK; ++tk)
      if (kind[tk] == 1) acc[tk] = sacc[tk];
  }
#pragma unroll
  for (int tk = 0; tk < TOK; ++tk) {
    const int m = m0 + tk;
    float v = 0.f;
    if (kind[tk] == 2) v = acc[tk] + p.temb[kbr[tk] * p.W + n];
    else if (kind[tk] == 1) v = acc[tk];
    p.x[(size_t)m * p.W + n] = v;
    p.xb[(size_t)m * p.W + n] = __float2bfloat16_rn(v);
    float sq = v * v;
    for (int off = 16; off; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (lane == 0) red[warp][tk] = sq;
  }
  __syncthreads();
  // per-128-feature-group sum of squares: warps 0-3 cover group 2y, 4-7 group 2y+1
  if (threadIdx.x < 2 * TOK) {
    const int half = threadIdx.x / TOK, tk = threadIdx.x % TOK;
    const float s = ((red[4 * half][tk] + red[4 * half + 1][tk]) + red[4 * half + 2][tk]) +
                    red[4 * half + 3][tk];
    p.ssq[(size_t)(2 * blockIdx.y + half) * p.ssq_ld + m0 + tk] = s;
  }
  if (threadIdx.x == 0) sm100::pdl_launch_dependents();
}

// [rows][cols] -> [cols][rows] of 8-byte elements (RoPE table, once per handle)
__global__ void transpose_u64_kernel(const unsigned long long* __restrict__ src,
                                     unsigned long long* __restrict__ dst, int rows, int cols) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * cols; i += gridDim.x * blockDim.x) {
    const int r = i / cols, c = i - r * cols;
    dst[(size_t)c * rows + r] = src[i];
  }
}

// Prefix K / V^T pool -> per-key-block SMEM images (SWIZZLE_128B, the layout
// TMA would write): K block j of (layer, env) = 4 chunks of [64 keys][64 dims],
// 16 B unit u of row r stored at unit (u ^ (r & 7)); V^T block = [256 dims][64
// keys] likewise by dim row. Keys >= P are zero. One thread per 16 B unit.
__global__ void prefix_image_kernel(const bf16* __restrict__ kp, const bf16* __restrict__ vp,
                                    uint8_t* __restrict__ kimg, uint8_t* __restrict__ vimg, int LE,
                                    int P, int nblk) {
  const size_t units_per_blk = 32768 / 16;  // 2048
  const size_t total = (size_t)LE * nblk * units_per_blk;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t le = i / (nblk * units_per_blk);
    const int rem = (int)(i - le * nblk * units_per_blk);
    const int j = rem / (int)units_per_blk, u = rem % (int)units_per_blk;
    // destination unit u -> (row, swizzled column unit)
    {  // K: chunk c (dims c*64..), row = key kk, unit position w holds column unit w ^ (kk & 7)
      const int c = u >> 9, rr = (u >> 3) & 63, w = u & 7;
      const int cu = w ^ (rr & 7);
      const int key = j * 64 + rr, d0 = c * 64 + cu * 8;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (key < P) v = *reinterpret_cast<const uint4*>(kp + ((size_t)le * P + key) * 256 + d0);
      reinterpret_cast<uint4*>(kimg + ((size_t)le * nblk + j) * 32768)[u] = v;
    }
    {  // V^T: row = dim (256 rows of 128 B), unit position w holds key unit w ^ (dim & 7)
      const int dim = u >> 3, w = u & 7;
      const int cu = w ^ (dim & 7);
      const int key0 = j * 64 + cu * 8;
      uint4 v = make_uint4(0, 0, 0, 0);
      const bf16* src = vp + ((size_t)le * 256 + dim) * P + key0;
      if (key0 + 8 <= P && (P % 8) == 0) {
        v = *reinterpret_cast<const uint4*>(src);
      } else {
        bf16 t[8];
        for (int z = 0; z < 8; ++z) t[z] = key0 + z < P ? src[z] : __float2bfloat16_rn(0.f);
        v = *reinterpret_cast<const uint4*>(t);
      }
      reinterpret_cast<uint4*>(vimg + ((size_t)le * nblk + j) * 32768)[u] = v;
    }
  }
}

// [rows][cols] -> [cols][rows] (embedding weights, once per handle)
__global__ void transpose_f32_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                     int rows, int cols) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * cols; i += gridDim.x * blockDim.x) {
    const int r = i / cols, c = i - r * cols;
    dst[(size_t)c * rows + r] = src[i];
  }
}

// --------------------------------------------------------- verify epilogue

struct VerifyEpiParams {
  int H, D, C, K, T, env_rows;
  float taus[SF_MAX_K];
  float delta;
  int metric, window;
  float sign;
  const float* signs;  // [B] or null
  int phase_fallback, prefix_cap, replan_size;
  const float* draft;  // [B][H][D]
  const float* eps;    // [B][H][D]
  const float* vel;    // [M][D] head output
  float* out_recon;    // [B][K][H][D] or null
  float* out_dist;     // [B][K][H] or null
  int* out_branch;     // [B][K]
  int* out_result;     // [B][8]
};

__global__ void __launch_bounds__(1024) verify_epi_kernel(const VerifyEpiParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  sm100::pdl_wait();
  const int e = blockIdx.x;
  float* s_recon = reinterpret_cast<float*>(smem_raw);
  float* s_dist = s_recon + p.K * p.H * p.D;
  const int HD = p.H * p.D;
  const float* vel = p.vel + (size_t)e * p.env_rows * p.D;
  verify_epilogue_cta<float, false>(
      p.draft + (size_t)e * HD, p.eps + (size_t)e * HD,
      [&](int k, int i) { return vel[(size_t)(k * p.T + 1) * p.D + i]; }, p.H, p.D, p.C, p.K,
      p.taus, p.delta, p.metric, p.window, p.signs ? p.signs[e] : p.sign, p.phase_fallback,
      p.prefix_cap, p.replan_size, p.out_recon ? p.out_recon + (size_t)e * p.K * HD : nullptr,
      p.out_dist ? p.out_dist + (size_t)e * p.K * p.H : nullptr, p.out_branch + e * p.K,
      p.out_result + e * SF_RESULT_WORDS, s_recon, s_dist);
}

struct EulerParams {
  float* A;
  const float* vel;
  int B, H, D, env_rows, n, step;
  int* status;
};

// A <- A + v / N with the finite check (flowpolicy.py:289-291), rows of the
// single-branch Euler layout (token 1 + h of env e).
__global__ void euler_rows_kernel(const EulerParams p) {
  sm100::pdl_wait();
  const int total = p.B * p.H * p.D;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int e = i / (p.H * p.D);
    const int rem = i - e * p.H * p.D;
    const int h = rem / p.D, d = rem - h * p.D;
    const float v = p.vel[((size_t)e * p.env_rows + 1 + h) * p.D + d];
    const float nxt = __fadd_rn(p.A[i], __fdiv_rn(v, (float)p.n));
    p.A[i] = nxt;
    if (!isfinite(v)) atomicCAS(&p.status[2 * e + 1], 0, 1);
    if (!isfinite(nxt)) atomicCAS(&p.status[2 * e], -1, p.step);
  }
  if (threadIdx.x == 0) sm100::pdl_launch_dependents();
}

struct SleepParams {
  long long ns;
};

__global__ void sleep_kernel(const SleepParams p) {
  const long long t0 = clock64();
  while (clock64() - t0 < p.ns * 2) __nanosleep(1000);
}

struct StatusParams {
  int* status;
  int B;
};

// Several small device copies / fills of 32-bit words in ONE launch (copy j
// = blockIdx.y; src == nullptr fills with fill[j]): the per-call staging of a
// speculative round was 4 input + 5 output cudaMemcpyAsync nodes at ~2 us of
// GPU time each around the graph.
struct CopyList {
  static constexpr int kMax = 10;
  const void* src[kMax];
  void* dst[kMax];
  long long n[kMax];  // 32-bit words
  float fill[kMax];
  int count;
};

__global__ void copy_list_kernel(const CopyList cl) {
  const int j = blockIdx.y;
  const uint32_t* src = static_cast<const uint32_t*>(cl.src[j]);
  uint32_t* dst = static_cast<uint32_t*>(cl.dst[j]);
  const long long n = cl.n[j];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  if (!src) {
    const uint32_t v = __float_as_uint(cl.fill[j]);
    for (long long i = tid; i < n; i += nt) dst[i] = v;
    return;
  }
  long long done = 0;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const long long n4 = n >> 2;
    for (long long i = tid; i < n4; i += nt)
      reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
    done = n4 << 2;
  }
  for (long long i = done + tid; i < n; i += nt) dst[i] = __ldg(src + i);
}

static void copy_list_add(CopyList& cl, void* dst, const void* src, long long words, float fill = 0.f) {
  cl.dst[cl.count] = dst;
  cl.src[cl.count] = src;
  cl.n[cl.count] = words;
  cl.fill[cl.count] = fill;
  ++cl.count;
}

static int copy_list_launch(const CopyList& cl, cudaStream_t s) {
  if (cl.count == 0) return SF_OK;
  long long mx = 1;
  for (int j = 0; j < cl.count; ++j) mx = cl.n[j] > mx ? cl.n[j] : mx;
  const long long blocks = (mx / 4 + 255) / 256;
  dim3 grid((unsigned)(blocks < 1 ? 1 : (blocks > 296 ? 296 : blocks)), (unsigned)cl.count);
  copy_list_kernel<<<grid, 256, 0, s>>>(cl);
  SF_CHECK_CUDA(cudaGetLastError());
  sf::count_launch();
  return SF_OK;
}

__global__ void status_init_kernel(const StatusParams p) {
  for (int e = threadIdx.x; e < p.B; e += blockDim.x) {
    p.status[2 * e] = -1;
    p.status[2 * e + 1] = 0;
  }
}

struct CastParams {
  const float* src;
  bf16* dst;
  int n;
};

// obs f32 -> bf16 GEMM operand (draft MLP input).
__global__ void cast_bf16_kernel(const CastParams p) {
  sm100::pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += gridDim.x * blockDim.x)
    p.dst[i] = __float2bfloat16_rn(p.src[i]);
  if (threadIdx.x == 0) sm100::pdl_launch_dependents();
}

struct GatherParams {
  const float* vel;
  float* out;  // [B][K][H][D]
  int B, K, H, D, T, env_rows;
};

__global__ void gather_vel_kernel(const GatherParams p) {
  const int total = p.B * p.K * p.H * p.D;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int d = i % p.D;
    const int h = (i / p.D) % p.H;
    const int k = (i / (p.D * p.H)) % p.K;
    const int e = i / (p.D * p.H * p.K);
    p.out[i] = p.vel[((size_t)e * p.env_rows + k * p.T + 1 + h) * p.D + d];
  }
}

// ------------------------------------------------- batched replanning round

constexpr int kMaxBuckets = 32;

struct ReplanSelectParams {
  int n;
  const int* result;
  int* fsr;
  int* has_cache;
  int mode_flash, pf, r;
  int* path;
  int* planned;
  int* fb_idx;
  int* fb_count;
  int n_buckets;
  int bucket[kMaxBuckets];
  cudaGraphConditionalHandle cond;
};

// round bookkeeping + compaction (replan.cuh), then the SWITCH value: the
// smallest pre-captured Euler bucket that holds the fallback envs (n_buckets
// = no full path this round)
__global__ void __launch_bounds__(1024) replan_select_kernel(const ReplanSelectParams p) {
  const int cnt = replan_update_cta(p.n, p.result, p.fsr, p.has_cache, p.mode_flash, p.pf, p.r, p.path,
                                    p.planned, p.fb_idx);
  if (threadIdx.x == 0) {
    *p.fb_count = cnt;
    unsigned sel = (unsigned)p.n_buckets;
    for (int i = 0; i < p.n_buckets && cnt > 0; ++i)
      if (cnt <= p.bucket[i]) {
        sel = (unsigned)i;
        break;
      }
    cudaGraphSetConditional(p.cond, sel);
  }
}

struct FlashSelectParams {
  int n;
  const int* fsr;
  const int* has_cache;
  int mode_flash, pf;
  int* use;       // [n] 1 = the env makes a flash attempt this round
  int* fl_idx;    // [n] attempting envs in env order
  int* fl_count;  // [1]
  int n_buckets;
  int bucket[kMaxBuckets];
  cudaGraphConditionalHandle cond;
};

// Which envs make a flash attempt this round (runtime.py:242-253: a cached
// context and no forced periodic refresh), compacted in env order; the SWITCH
// value is the smallest pre-captured flash bucket holding them (n_buckets =
// none: a round of full rounds only runs no speculative attempt at all).
__global__ void __launch_bounds__(1024) flash_select_kernel(const FlashSelectParams p) {
  __shared__ int warp_tot[32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < p.n; c0 += blockDim.x) {
    const int e = c0 + tid;
    int u = 0;
    if (e < p.n) {
      const bool forced = p.pf > 0 && p.fsr[e] >= p.pf;
      u = p.mode_flash && p.has_cache[e] && !forced;
      p.use[e] = u;
    }
    const unsigned m = __ballot_sync(0xffffffffu, u);
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
      int v = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      warp_tot[lane] = v;
    }
    __syncthreads();
    if (u) p.fl_idx[base + (warp ? warp_tot[warp - 1] : 0) + __popc(m & ((1u << lane) - 1u))] = e;
    __syncthreads();
    if (tid == 0) base += warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (tid == 0) {
    *p.fl_count = base;
    unsigned sel = (unsigned)p.n_buckets;
    for (int i = 0; i < p.n_buckets && base > 0; ++i)
      if (base <= p.bucket[i]) {
        sel = (unsigned)i;
        break;
      }
    cudaGraphSetConditional(p.cond, sel);
  }
}

// flash bucket row j <- attempting env fl_idx[j] (rows past the count repeat
// the first one; their results are dropped): observation, verify noise,
// state, sign and the env's prefix-KV slot
struct FlashGatherParams {
  const int* fl_idx;
  const int* fl_count;
  int Bk, F, HD, S;
  const float *obs, *eps, *state, *signs;
  float *obs_o, *eps_o, *state_o, *signs_o;
  int* env_map;
};

__global__ void flash_gather_kernel(const FlashGatherParams p) {
  const int cnt = *p.fl_count;
  const int per = p.F + p.HD + p.S + 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.Bk * per; i += gridDim.x * blockDim.x) {
    const int j = i / per;
    int c = i - j * per;
    const int e = p.fl_idx[j < cnt ? j : 0];
    if (c < p.F) {
      p.obs_o[(size_t)j * p.F + c] = p.obs[(size_t)e * p.F + c];
    } else if ((c -= p.F) < p.HD) {
      p.eps_o[(size_t)j * p.HD + c] = p.eps[(size_t)e * p.HD + c];
    } else if ((c -= p.HD) < p.S) {
      p.state_o[(size_t)j * p.S + c] = p.state[(size_t)e * p.S + c];
    } else {
      p.signs_o[j] = p.signs[e];
      p.env_map[j] = e;
    }
  }
}

// attempt results back to their envs: result words, branch prefixes, draft
struct FlashScatterParams {
  const int* fl_idx;
  const int* fl_count;
  int K, HD;
  const int *result, *branch;
  const float* draft;
  int *result_o, *branch_o;
  float* draft_o;
};

__global__ void flash_scatter_kernel(const FlashScatterParams p) {
  const int cnt = *p.fl_count;
  const int per = SF_RESULT_WORDS + p.K + p.HD;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt * per; i += gridDim.x * blockDim.x) {
    const int j = i / per;
    int c = i - j * per;
    const int e = p.fl_idx[j];
    if (c < SF_RESULT_WORDS) {
      p.result_o[e * SF_RESULT_WORDS + c] = p.result[j * SF_RESULT_WORDS + c];
    } else if ((c -= SF_RESULT_WORDS) < p.K) {
      p.branch_o[e * p.K + c] = p.branch[j * p.K + c];
    } else {
      c -= p.K;
      p.draft_o[(size_t)e * p.HD + c] = p.draft[(size_t)j * p.HD + c];
    }
  }
}

// envs without an attempt this round: result words 0..SF_RES_NONFINITE and branch prefixes -1
// (the reference's RoundRecord has no prefix / branch prefixes for them)
__global__ void flash_mark_kernel(const int* __restrict__ use, int n, int K, int* __restrict__ result,
                                  int* __restrict__ branch) {
  const int per = SF_RESULT_WORDS + K;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * per; i += gridDim.x * blockDim.x) {
    const int e = i / per, c = i - e * per;
    if (use[e]) continue;
    if (c < SF_RESULT_WORDS) {
      if (c <= SF_RES_NONFINITE) result[e * SF_RESULT_WORDS + c] = -1;  // reserved words untouched
    } else {
      branch[e * K + (c - SF_RESULT_WORDS)] = -1;
    }
  }
}

// chunk <- draft for every env (accepted envs execute it); clear the flags
__global__ void chunk_init_kernel(const float* __restrict__ draft, float* __restrict__ chunk,
                                  int* __restrict__ bad, int n, int hd) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * hd; i += gridDim.x * blockDim.x) {
    chunk[i] = draft[i];
    if (i < n) bad[i] = 0;
  }
}

// bucket row j <- fallback env fb_idx[j] (rows past the count repeat the
// first fallback env; their results are dropped)
__global__ void bucket_gather_kernel(const int* __restrict__ fb_idx, const int* __restrict__ fb_count, int Bk,
                                     int hd, int S, const float* __restrict__ eps_d,
                                     const float* __restrict__ state_in, float* __restrict__ start,
                                     float* __restrict__ state_out, int* __restrict__ env_map) {
  const int cnt = *fb_count;
  const int per = hd + S;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Bk * per; i += gridDim.x * blockDim.x) {
    const int j = i / per, c = i - j * per;
    const int e = fb_idx[j < cnt ? j : 0];
    if (c < hd) start[(size_t)j * hd + c] = eps_d[(size_t)e * hd + c];
    else state_out[(size_t)j * S + (c - hd)] = state_in[(size_t)e * S + (c - hd)];
    if (c == 0) env_map[j] = e;
  }
}

// full-path chunks back to their envs; Euler status -> non-finite flag
__global__ void bucket_scatter_kernel(const int* __restrict__ fb_idx, const int* __restrict__ fb_count,
                                      int hd, const float* __restrict__ A, const int* __restrict__ status,
                                      float* __restrict__ chunk, int* __restrict__ bad) {
  const int cnt = *fb_count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt * hd; i += gridDim.x * blockDim.x) {
    const int j = i / hd, c = i - j * hd;
    const int e = fb_idx[j];
    chunk[(size_t)e * hd + c] = A[i];
    if (c == 0) bad[e] = (status[2 * j] >= 0 || status[2 * j + 1]) ? 1 : 0;
  }
}

struct ReplanFinalParams {
  int n, H, D;
  const int* path;
  int* planned;
  const int* result;
  const float* signs;
  float* chunk;
  int* bad;
  int* sie;
  float* chunk_raw;
  const float* mean;
  const float* stdv;
};

// one warp per env: non-finite accepted chunks (actions.py:65-74 rejects them,
// verifier.py:89 raises on a non-finite reconstruction), switch_in_executed
// (runtime.py:321-323: gripper_switch(chunk[:planned], sign)), planned = 0 for
// a non-finite chunk, destandardize (actions.py:139-144: raw = z * std + mean)
__global__ void replan_finalize_kernel(const ReplanFinalParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= p.n) return;
  const int e = warp, hd = p.H * p.D;
  float* c = p.chunk + (size_t)e * hd;
  const bool acc = p.path[e] == SF_PATH_FLASH_ACCEPTED;
  int bad = p.bad[e];
  if (acc) {
    bool nf = p.result[e * SF_RESULT_WORDS + SF_RES_NONFINITE] >= 0;
    for (int i = lane; i < hd; i += 32) nf |= !isfinite(c[i]);
    bad = __any_sync(0xffffffffu, nf) ? 1 : 0;
  }
  const int pl = p.planned[e];
  int sw = 0;
  if (acc && !bad) {
    const float sg = p.signs[e];
    bool hit = false;
    for (int h = lane; h < pl; h += 32) hit |= c[(size_t)h * p.D + p.D - 1] * sg <= 0.f;
    sw = __any_sync(0xffffffffu, hit) ? 1 : 0;
  }
  if (lane == 0) {
    p.bad[e] = bad;
    p.sie[e] = sw;
    if (bad) p.planned[e] = 0;
  }
  if (p.chunk_raw)
    for (int i = lane; i < hd; i += 32) {
      const int d = i % p.D;
      p.chunk_raw[(size_t)e * hd + i] = __fadd_rn(__fmul_rn(c[i], p.stdv[d]), p.mean[d]);
    }
}

// ----------------------------------------------------------------- handle

struct Buffers {
  int B = 0, K = 0, env_rows = 0, M = 0, m_ld = 0;
  float* x = nullptr;      // [M][W]
  bf16* xb = nullptr;      // [M][W]
  float* ssq = nullptr;    // [8][m_ld]
  bf16* q = nullptr;       // [M][8*256]
  bf16* ks = nullptr;      // [M][256]
  bf16* vt = nullptr;      // [256][m_ld]
  bf16* attn = nullptr;    // [M][8*256]
  bf16* h = nullptr;       // [M][mlp]
  float* vel = nullptr;    // [M][D]
  float* draft = nullptr;  // [B][H][D] staged inputs (graph-stable)
  float* eps = nullptr;
  float* state = nullptr;  // [B][S]
  float* signs = nullptr;  // [B]
  float* recon = nullptr;  // [B][K][H][D]
  float* dist = nullptr;   // [B][K][H]
  int* branch = nullptr;   // [B][K]
  int* result = nullptr;   // [B][8]
  int* status = nullptr;   // [B][2] Euler status
  int* env_map = nullptr;  // [B] prefix-KV pool slot per batch env (read by attention)
  int* env_ident = nullptr;  // [B] identity map
  float* ws = nullptr;
  size_t ws_bytes = 0;
  int* counters = nullptr;
  int n_counters = 0;
  std::vector<gemm::Op> ops;     // per layer: qkv, o, gu, down; then head
  std::vector<size_t> attn_ops;  // unused placeholder
  attn::Params ap{};
  int attn_tiles = 0, attn_splits = 1;
  std::vector<CUtensorMap> attn_maps;  // per layer: q, kp, vp, ks, vs
  std::vector<CUtensorMap> attn_pair_maps;  // 2-SM pair kernel: half-block boxes (batched)
  bool attn_pair = false;
  const uint8_t* k_img = nullptr;  // handle's prefix block images (null: tensor maps)
  const uint8_t* v_img = nullptr;
  int img_blocks = 0, n_img_envs = 0;
  cudaGraphExec_t graph = nullptr;
  int graph_key = 0;
  int graph_kernels = 0;  // kernel nodes in `graph` (launch accounting)
  // draft MLP (flash rounds)
  float* obs = nullptr;   // [B][F]
  bf16* obs_b = nullptr;  // [b_ld][F]
  bf16* dh1 = nullptr;    // [b_ld][hidden]
  bf16* dh2 = nullptr;
  gemm::Op dops[3];
  bool has_draft = false;
  // fp32 mode (SF_AE_FP32): fp32 activations of the CUDA-core layer stack
  bool fp32 = false;
  float* f_rs = nullptr;   // [M] RMS row scales
  float* f_qkv = nullptr;  // [M][(nh + 2) * 256] device row order
  float* f_q = nullptr;    // [M][nh * 256]
  float* f_k = nullptr;    // [M][256]
  float* f_v = nullptr;    // [M][256]
  float* f_o = nullptr;    // [M][nh * 256]
  float* f_gu = nullptr;   // [M][2 * mlp]
  float* f_h = nullptr;    // [M][mlp]
};

struct Handle {
  int replan_kernels[4] = {0, 0, 0, 0};  // last replanning round: fixed, flash verify, Euler body, max sub-n flash bucket
  sf_ae_config_t cfg{};
  sf_ae_weights_t w{};
  const bf16* k_prefix = nullptr;   // [L][E][P][256]
  const bf16* vt_prefix = nullptr;  // [L][E][256][P]
  int n_prefix_envs = 0;
  float* temb = nullptr;   // [SF_MAX_K][W] for the verify taus
  float temb_taus[SF_MAX_K];
  int temb_k = -1;
  float* temb_euler = nullptr;  // [N][W]
  int temb_euler_n = -1;
  float* temb_hidden = nullptr;
  float* temb_tau_dev = nullptr;
  float* a_wt = nullptr;  // [D][W] transposed action-embedding weights
  float* s_wt = nullptr;  // [S][W] transposed state-embedding weights
  float2* rope_t = nullptr;  // [head_dim/2][P + 1 + H] position-fastest RoPE table
  uint8_t* k_img = nullptr;  // [L][E][nblk][32 KB] prefix K block images (attention)
  uint8_t* v_img = nullptr;  // [L][E][nblk][32 KB] prefix V^T block images
  int img_blocks = 0;
  std::map<long long, std::unique_ptr<Buffers>> buffers;  // key: (B, K, mode)
  std::map<uint64_t, std::unique_ptr<struct Replan>> replans;
  cudaStream_t capture_stream = nullptr;
  cudaStream_t body_stream = nullptr;  // conditional-body captures
  struct B1Engine* b1 = nullptr;       // persistent batch-1 Euler engine (lazy)
};

// Graph-resident replanning round (sf_ae_replan_round): owned device buffers
// and the instantiated graph for one (n, cfg, policy, state pointers) key.
struct Replan {
  int n = 0, K = 0;
  Buffers* bf = nullptr;             // flash buffers (B = n, K)
  std::vector<int> buckets;          // Euler bucket sizes
  std::vector<Buffers*> bb;          // denoise buffers per bucket
  float* eps_d = nullptr;            // [n][H][D] staged denoise noise
  float* chunk = nullptr;            // [n][H][D]
  float* chunk_raw = nullptr;        // [n][H][D]
  float* mean = nullptr;             // [D]
  float* stdv = nullptr;             // [D]
  int *path = nullptr, *planned = nullptr, *sie = nullptr, *bad = nullptr;
  int *fb_idx = nullptr, *fb_count = nullptr;
  std::vector<int> fbuckets;         // flash-attempt bucket sizes (the last one = n runs on bf)
  std::vector<Buffers*> fbb;         // verify buffers per flash bucket (nullptr for n: bf)
  int *use = nullptr, *fl_idx = nullptr, *fl_count = nullptr;
  cudaGraphExec_t exec = nullptr;
  int fixed_kernels = 0;             // kernels of a round with neither an attempt nor the full path
  int flash_body_kernels = 0;        // kernels of a compacted flash-attempt body (the n-env body: 2 fewer)
  int euler_body_kernels = 0;        // kernels of an Euler bucket body
  ~Replan() {
    if (exec) cudaGraphExecDestroy(exec);
    for (void* q : {(void*)eps_d, (void*)chunk, (void*)chunk_raw, (void*)mean, (void*)stdv, (void*)path,
                    (void*)planned, (void*)sie, (void*)bad, (void*)fb_idx, (void*)fb_count, (void*)use,
                    (void*)fl_idx, (void*)fl_count})
      if (q) cudaFree(q);
  }
};

int T_of(const Handle& h) { return 1 + h.cfg.horizon; }

template <typename P>
int launch_pdl(void (*kern)(P), dim3 grid, dim3 block, size_t smem, cudaStream_t s, const P& p,
               bool pdl) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
  count_launch();
  return SF_OK;
}

// 8 token rows per CTA for batched rounds (lighter CTAs: 48 registers, more resident), else 16
int launch_embed(int M, int W, cudaStream_t s, const EmbedParams& ep, bool pdl) {
  if (M % 8 == 0 && M >= 148 * 64) return launch_pdl(embed_kernel<8>, dim3(M / 8, W / 256), dim3(256), 0, s, ep, pdl);
  return launch_pdl(embed_kernel<kEmbedTok>, dim3(M / kEmbedTok, W / 256), dim3(256), 0, s, ep, pdl);
}

int compute_temb(Handle& h, const float* taus_host, int R, float* out, cudaStream_t s) {
  const int W = h.cfg.width;
  SF_CHECK_CUDA(cudaMemcpyAsync(h.temb_tau_dev, taus_host, sizeof(float) * R,
                                cudaMemcpyHostToDevice, s));
  const size_t smem = sizeof(float) * R * W;
  SF_REQUIRE(smem <= 200 * 1024, "too many taus for the time embedding (%d)", R);
  SF_CHECK_CUDA(cudaFuncSetAttribute(temb_hidden_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  temb_hidden_kernel<<<64, 256, smem, s>>>((const float*)h.w.t1_w, (const float*)h.w.t1_b,
                                           h.temb_tau_dev, R, W, h.cfg.temb_min_period,
                                           h.cfg.temb_max_period, h.temb_hidden);
  temb_out_kernel<<<64, 256, 0, s>>>((const float*)h.w.t2_w, (const float*)h.w.t2_b,
                                     h.temb_hidden, R, W, out);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch(2);
  return SF_OK;
}

int make_map_3d(CUtensorMap* m, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2,
                uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("3-D tensor map encode failed (%d)", (int)r);
    return SF_ECUDA;
  }
  return SF_OK;
}

template <typename T>
int dalloc(T** p, size_t n) {
  SF_CHECK_CUDA(cudaMalloc(p, sizeof(T) * (n ? n : 1)));
  SF_CHECK_CUDA(cudaMemset(*p, 0, sizeof(T) * (n ? n : 1)));
  return SF_OK;
}

// Build buffers + GEMM / attention plans for B envs x K branches.
int build(Handle& h, Buffers& b, int B, int K) {
  const sf_ae_config_t& c = h.cfg;
  const int W = c.width, T = T_of(h), L = c.layers;
  const int nq = c.q_heads * c.head_dim;
  b.B = B;
  b.K = K;
  // dense env rows (no per-env padding: the GEMMs see only real tokens; the
  // attention's 16-token query tiles restart at every env), rows padded to a
  // multiple of 16 at the end of the batch
  b.env_rows = K * T;
  b.M = ((B * b.env_rows + 15) / 16) * 16;
  b.m_ld = ((b.M + 63) / 64) * 64;
  int rc;
#define ALLOC(ptr, n) \
  if ((rc = dalloc(&(ptr), (n)))) return rc
  ALLOC(b.x, (size_t)b.M * W);
  ALLOC(b.xb, (size_t)b.m_ld * W);
  ALLOC(b.ssq, (size_t)(W / 128) * b.m_ld);
  ALLOC(b.q, (size_t)b.m_ld * nq);
  ALLOC(b.ks, (size_t)b.m_ld * c.head_dim);
  ALLOC(b.vt, (size_t)c.head_dim * b.m_ld);
  ALLOC(b.attn, (size_t)b.m_ld * nq);
  ALLOC(b.h, (size_t)b.m_ld * c.mlp);
  ALLOC(b.vel, (size_t)b.M * c.action_dim);
  ALLOC(b.draft, (size_t)B * c.horizon * c.action_dim);
  ALLOC(b.eps, (size_t)B * c.horizon * c.action_dim);
  ALLOC(b.state, (size_t)B * c.state_dim);
  ALLOC(b.signs, (size_t)B);
  ALLOC(b.recon, (size_t)B * K * c.horizon * c.action_dim);
  ALLOC(b.dist, (size_t)B * K * c.horizon);
  ALLOC(b.branch, (size_t)B * K);
  ALLOC(b.result, (size_t)B * SF_RESULT_WORDS);
  ALLOC(b.status, (size_t)B * 2);
  ALLOC(b.env_map, (size_t)B);
  ALLOC(b.env_ident, (size_t)B);
  {
    std::vector<int> ident(B);
    for (int i = 0; i < B; ++i) ident[i] = i;
    SF_CHECK_CUDA(cudaMemcpy(b.env_ident, ident.data(), sizeof(int) * B, cudaMemcpyHostToDevice));
    SF_CHECK_CUDA(cudaMemcpy(b.env_map, ident.data(), sizeof(int) * B, cudaMemcpyHostToDevice));
  }
  const int b_ld = ((B + 63) / 64) * 64;
  b.has_draft = c.draft_in > 0 && h.w.draft_w[0] != nullptr;
  if (b.has_draft) {
    ALLOC(b.obs, (size_t)B * c.draft_in);
    ALLOC(b.obs_b, (size_t)b_ld * c.draft_in);
    ALLOC(b.dh1, (size_t)b_ld * c.draft_hidden);
    ALLOC(b.dh2, (size_t)b_ld * c.draft_hidden);
  }

  // --- GEMM plans. Batch-1 shapes stream weights (swap-AB + split-K);
  // larger batches run the normal orientation with 256-feature tiles.
  // Batch-1 shapes stream weights: swap-AB + split-K reduced over DSMEM in a
  // CTA cluster. Larger batches: persistent 128 x 256 tiles.
  const bool swap = b.M <= 256;
  const int bn_swap = ((b.M + 15) / 16) * 16;
  const int bn_norm = 256;
  const int bn_head = swap ? bn_swap : 32;
  int max_tiles = 0;
  // attention split-KV workspace
  const int n_prefix_blocks = (c.prefix_len + attn::BKEY - 1) / attn::BKEY;
  // suffix keys of the (<= 2) segments a 16-token tile touches, from a
  // 64-aligned start: span <= 63 + 2 * T
  const int n_blocks = n_prefix_blocks + (63 + 2 * T + attn::BKEY - 1) / attn::BKEY;
  const int tiles_env = (b.env_rows + 15) / 16;
  b.attn_tiles = B * tiles_env;
  int asplit = 148 / b.attn_tiles;
  if (getenv("SF_ATTN_SPLITS")) asplit = atoi(getenv("SF_ATTN_SPLITS"));  // debug override
  if (asplit < 1) asplit = 1;
  if (asplit > n_blocks) asplit = n_blocks;
  if (asplit > attn::kMaxSplitsKV) asplit = attn::kMaxSplitsKV;
  if (asplit > 8 && !getenv("SF_ATTN_SPLITS")) asplit = 8;  // merge traffic grows with the split count (Euler: 8 beats 16)
  const int bps = (n_blocks + asplit - 1) / asplit;
  asplit = (n_blocks + bps - 1) / bps;
  b.attn_splits = asplit;  // split-KV CTAs of a tile form one cluster (DSMEM merge)
  float* attn_ws = nullptr;
  if (asplit > 1) {
    // split-KV partials: [tiles][splits][HD/4][128] float4 + (m, l) [tiles][splits][128]
    const size_t n = (size_t)b.attn_tiles * asplit * (attn::HD * attn::BQ + 2 * attn::BQ);
    if ((rc = dalloc(&attn_ws, n))) return rc;
  }
  b.n_counters = (max_tiles > b.attn_tiles ? max_tiles : b.attn_tiles) + 8;
  ALLOC(b.counters, (size_t)b.n_counters);
#undef ALLOC

  auto epi_base = [&](int kind) {
    gemm::EpiArgs e{};
    e.kind = kind;
    e.M = b.M;
    e.ssq_in = b.ssq;
    e.ssq_groups = W / 128;
    e.ssq_ld = b.m_ld;
    e.inv_width = 1.f / (float)W;
    e.eps = c.eps;
    return e;
  };
  b.ops.resize(4 * L + 1);
  // token rows `rows` (activations, K-major) x weights [n_out, k_in]
  auto plan_mm = [&](gemm::Op* op, const void* wt, int n_out, const void* act, int rows, int k_in,
                     int bn, bool sw, const gemm::EpiArgs& e) {
    if (sw) return gemm::plan(op, wt, n_out, k_in, act, rows, k_in, k_in, bn, 0, 1, e);
    return gemm::plan(op, act, rows, k_in, wt, n_out, k_in, k_in, bn, 1, 0, e);
  };
  int nsm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  struct Spec {
    const void* wt;
    int n_out;
    const void* act;
    int k_in;
    gemm::EpiArgs e;
  };
  std::vector<Spec> specs(4 * L);
  auto plan_op = [&](gemm::Op* op, const void* wt, int n_out, const void* act, int k_in,
                     const gemm::EpiArgs& e) {
    const int idx = (int)(op - b.ops.data());
    if (idx < 4 * L) specs[idx] = Spec{wt, n_out, act, k_in, e};
    return plan_mm(op, wt, n_out, act, b.M, k_in, swap ? bn_swap : bn_norm, swap, e);
  };
  for (int l = 0; l < L; ++l) {
    gemm::EpiArgs e = epi_base(gemm::EPI_QKV);
    e.N = nq + 2 * c.head_dim;
    e.q = b.q;
    e.k = b.ks;
    e.vt = b.vt;
    e.vt_ld = b.m_ld;
    e.rope = h.rope_t;
    e.rope_ld = c.prefix_len + 1 + c.horizon;
    e.q_features = nq;
    e.env_rows = b.env_rows;
    e.seg_len = T;
    e.pos0 = c.prefix_len;
    if ((rc = plan_op(&b.ops[4 * l + 0], h.w.qkv[l], e.N, b.xb, W, e))) return rc;
    gemm::EpiArgs eo = epi_base(gemm::EPI_RESID);
    eo.ssq_in = nullptr;
    eo.N = W;
    eo.x = b.x;
    eo.xb = b.xb;
    eo.ssq_out = b.ssq;
    eo.ssq_out_ld = b.m_ld;
    if ((rc = plan_op(&b.ops[4 * l + 1], h.w.o[l], W, b.attn, nq, eo))) return rc;
    gemm::EpiArgs eg = epi_base(gemm::EPI_GEGLU);
    eg.N = 2 * c.mlp;
    eg.out_bf16 = b.h;
    eg.ld_bf16 = c.mlp;
    if ((rc = plan_op(&b.ops[4 * l + 2], h.w.gu[l], eg.N, b.xb, W, eg))) return rc;
    if ((rc = plan_op(&b.ops[4 * l + 3], h.w.down[l], W, b.h, c.mlp, eo))) return rc;
  }
  {
    gemm::EpiArgs e = epi_base(gemm::EPI_F32);
    e.N = c.action_dim;
    e.out_f32 = b.vel;
    e.ld_f32 = c.action_dim;
    e.bias = static_cast<const float*>(h.w.out_b);
    if ((rc = plan_mm(&b.ops[4 * L], h.w.out_w, c.action_dim, b.xb, b.M, W, bn_head, swap, e)))
      return rc;
  }
  // --- draft MLP plans: rows = envs (swap-AB while B <= 256)
  if (b.has_draft) {
    const bool dswap = B <= 256;
    const int dbn = dswap ? ((B + 15) / 16) * 16 : 256;
    const int HDc = c.horizon * c.action_dim;
    const void* ins[3] = {b.obs_b, b.dh1, b.dh2};
    const int kin[3] = {c.draft_in, c.draft_hidden, c.draft_hidden};
    const int nout[3] = {c.draft_hidden, c.draft_hidden, HDc};
    bf16* outs[2] = {b.dh1, b.dh2};
    for (int i = 0; i < 3; ++i) {
      gemm::EpiArgs e{};
      e.kind = i < 2 ? gemm::EPI_TANH_BF16 : gemm::EPI_F32;
      e.M = B;
      e.N = nout[i];
      e.bias = static_cast<const float*>(h.w.draft_b[i]);
      if (i < 2) {
        e.out_bf16 = outs[i];
        e.ld_bf16 = c.draft_hidden;
      } else {
        e.out_f32 = b.draft;
        e.ld_f32 = HDc;
      }
      if ((rc = plan_mm(&b.dops[i], h.w.draft_w[i], nout[i], ins[i], B, kin[i], dbn, dswap, e)))
        return rc;
    }
  }
  // --- batch-1 plan tuning: the swap-AB GEMMs trade K splits (fp32 partials
  // through L2) against token tiles (weights re-read from L2); the best mix
  // depends on the token count, so each layer GEMM class (qkv, o, gu, down --
  // identical across layers) is timed over a small (bn, splits) grid on this
  // device and every layer is re-planned with the winner.
  // Default (deterministic across processes): a static rule distilled from the
  // measured (bn, splits) sweeps (scripts/gemm_sweep.py sweep): above 128
  // token rows use two token tiles (weights re-read from L2 beat fp32 partials),
  // then as many K splits as keep one wave with clusters <= 6 CTAs (8- and
  // 16-CTA clusters schedule poorly). SF_TUNE=1 times candidates instead.
  if (swap && getenv("SF_TUNE") == nullptr) {
    // SF_B1_PLAN="bn:S,bn:S,bn:S,bn:S" (qkv, o, gu, down; 0 = the rule's
    // value) overrides the rule for batches above 128 rows: the in-graph
    // sweep (scripts/b1_plan_sweep.py) times whole verify rounds with it
    int force_bn[4] = {0, 0, 0, 0}, force_s[4] = {0, 0, 0, 0};
    if (const char* fp = getenv("SF_B1_PLAN")) {
      if (b.M > 128)
        sscanf(fp, "%d:%d,%d:%d,%d:%d,%d:%d", &force_bn[0], &force_s[0], &force_bn[1], &force_s[1], &force_bn[2],
               &force_s[2], &force_bn[3], &force_s[3]);
    }
    for (int cls = 0; cls < 4; ++cls) {
      const Spec& sp = specs[cls];
      const int bn = force_bn[cls] > 0 ? force_bn[cls] : (b.M > 128 ? (((b.M + 1) / 2 + 15) / 16) * 16 : bn_swap);
      const int tiles_b = (b.M + bn - 1) / bn;
      const int tiles = ((sp.n_out + gemm::BM - 1) / gemm::BM) * tiles_b, nkb = sp.k_in / gemm::BK;
      int S = nsm / tiles;
      // 8-CTA clusters only while they fill at most half the GPU
      S = S > 8 ? 8 : (S < 1 ? 1 : S);
      if (S > 6 && tiles * S > nsm / 2) S = 6;
      S = S > nkb ? nkb : S;
      if (force_s[cls] > 0) S = force_s[cls];
      for (int l = 0; l < L; ++l) {
        const Spec& q = specs[4 * l + cls];
        if ((rc = gemm::plan(&b.ops[4 * l + cls], q.wt, q.n_out, q.k_in, q.act, b.M, q.k_in, q.k_in,
                             bn, S, 1, q.e)))
          return rc;
      }
    }
  } else if (swap && getenv("SF_NO_TUNE") == nullptr) {
    cudaStream_t ts;
    SF_CHECK_CUDA(cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    SF_CHECK_CUDA(cudaEventCreate(&e0));
    SF_CHECK_CUDA(cudaEventCreate(&e1));
    float* tws = nullptr;
    size_t tws_bytes = 0;
    auto c16 = [](int x) { return ((x + 15) / 16) * 16; };
    // decisions are cached per (shape, rows) for the process: every handle of
    // the same shape then runs the same plan (bitwise-identical results)
    static std::map<std::tuple<int, int, int, int>, std::pair<int, int>> tuned;
    for (int cls = 0; cls < 4; ++cls) {
      const Spec& sp = specs[cls];
      const auto key = std::make_tuple(sp.n_out, sp.k_in, b.M, sp.e.kind);
      auto hit = tuned.find(key);
      if (hit != tuned.end()) {
        for (int l = 0; l < L; ++l) {
          const Spec& q = specs[4 * l + cls];
          if ((rc = gemm::plan(&b.ops[4 * l + cls], q.wt, q.n_out, q.k_in, q.act, b.M, q.k_in,
                               q.k_in, hit->second.first, hit->second.second, 1, q.e)))
            return rc;
        }
        continue;
      }
      const int tiles_a = (sp.n_out + gemm::BM - 1) / gemm::BM, nkb = sp.k_in / gemm::BK;
      int bns[4] = {bn_swap, c16((b.M + 1) / 2), 64, 32};
      float best = 1e30f;
      int best_bn = bn_swap, best_s = 0;
      for (int bi = 0; bi < 4; ++bi) {
        const int bn = bns[bi];
        bool dup = bn > bn_swap;
        for (int bj = 0; bj < bi; ++bj) dup = dup || bns[bj] == bn;
        if (dup) continue;
        const int tiles = tiles_a * ((b.M + bn - 1) / bn);
        const int Ss[6] = {1, 2, 3, 4, 6, 8};
        for (int S : Ss) {
          if (S > nkb || (S > 1 && tiles * S > nsm)) continue;
          gemm::Op op;
          if (gemm::plan(&op, sp.wt, sp.n_out, sp.k_in, sp.act, b.M, sp.k_in, sp.k_in, bn, S, 1, sp.e))
            continue;
          if (op.p.splits != S) continue;  // K does not split that way
          if (op.ws_bytes > tws_bytes) {
            if (tws) cudaFree(tws);
            SF_CHECK_CUDA(cudaMalloc(&tws, op.ws_bytes));
            tws_bytes = op.ws_bytes;
          }
          op.p.ws = tws;
          // serialised launches (no PDL): with PDL, back-to-back copies of
          // the same GEMM overlap and reward configs that leave SMs idle
          for (int i = 0; i < 3; ++i)
            if ((rc = gemm::launch(op, ts, false))) return rc;
          SF_CHECK_CUDA(cudaEventRecord(e0, ts));
          for (int i = 0; i < 20; ++i)
            if ((rc = gemm::launch(op, ts, false))) return rc;
          SF_CHECK_CUDA(cudaEventRecord(e1, ts));
          SF_CHECK_CUDA(cudaEventSynchronize(e1));
          float ms = 0.f;
          cudaEventElapsedTime(&ms, e0, e1);
          if (getenv("SF_TUNE_VERBOSE"))
            printf("tune cls %d (N=%d K=%d M=%d): bn=%d S=%d grid=(%d,%d,%d) %.2f us\n", cls, sp.n_out,
                   sp.k_in, b.M, bn, S, op.grid.x, op.grid.y, op.grid.z, ms * 50.f);
          if (ms < best * 0.98f) best = ms, best_bn = bn, best_s = S;
        }
      }
      tuned[key] = std::make_pair(best_bn, best_s);
      for (int l = 0; l < L; ++l) {
        const Spec& q = specs[4 * l + cls];
        if ((rc = gemm::plan(&b.ops[4 * l + cls], q.wt, q.n_out, q.k_in, q.act, b.M, q.k_in, q.k_in,
                             best_bn, best_s, 1, q.e)))
          return rc;
      }
    }
    if (tws) cudaFree(tws);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(ts);
  }
  // --- one split-K workspace shared by every GEMM (kernels are stream-ordered;
  // with PDL a GEMM only touches it after griddepcontrol.wait)
  {
    size_t need = 0;
    for (auto& op : b.ops) need = op.ws_bytes > need ? op.ws_bytes : need;
    if (b.has_draft)
      for (auto& op : b.dops) need = op.ws_bytes > need ? op.ws_bytes : need;
    b.ws_bytes = need;
    if (need) {
      if ((rc = dalloc(&b.ws, need / sizeof(float)))) return rc;
      for (auto& op : b.ops) op.p.ws = b.ws;
      if (b.has_draft)
        for (auto& op : b.dops) op.p.ws = b.ws;
    }
  }
  // --- attention plans (per layer: 5 tensor maps)
  attn::Params& ap = b.ap;
  ap.M = B * b.env_rows;
  ap.env_rows = b.env_rows;
  ap.n_envs = B;
  ap.tiles_env = tiles_env;
  ap.seg_len = T;
  ap.segs = K;
  ap.prefix_len = c.prefix_len;
  ap.n_prefix_blocks = n_prefix_blocks;
  ap.n_blocks = n_blocks;
  ap.blocks_per_split = bps;
  ap.splits = asplit;
  ap.tiles = b.attn_tiles;
  ap.scale_log2 = 1.4426950408889634f / sqrtf((float)c.head_dim);
  ap.out = b.attn;
  ap.ws = attn_ws;
  ap.counters = b.counters;
  ap.env_map = b.env_map;
  b.k_img = h.k_img;
  b.v_img = h.v_img;
  b.img_blocks = h.img_blocks;
  b.n_img_envs = h.n_prefix_envs;  // shared with split-K GEMMs: kernels are stream-ordered
  b.attn_maps.resize(5 * L);
  const int E = h.n_prefix_envs;
  for (int l = 0; l < L; ++l) {
    CUtensorMap* mp = &b.attn_maps[5 * l];
    if ((rc = gemm::make_map(&mp[0], b.q, b.M * attn::kHeads, c.head_dim, c.head_dim, attn::BQ)))
      return rc;
    const bf16* kp = h.k_prefix + (size_t)l * E * c.prefix_len * c.head_dim;
    const bf16* vp = h.vt_prefix + (size_t)l * E * c.head_dim * c.prefix_len;
    if ((rc = make_map_3d(&mp[1], kp, c.head_dim, c.prefix_len, E, (uint64_t)c.head_dim * 2,
                          (uint64_t)c.prefix_len * c.head_dim * 2, 64, attn::BKEY)))
      return rc;
    if ((rc = make_map_3d(&mp[2], vp, c.prefix_len, c.head_dim, E, (uint64_t)c.prefix_len * 2,
                          (uint64_t)c.prefix_len * c.head_dim * 2, attn::BKEY, c.head_dim)))
      return rc;
    if ((rc = gemm::make_map(&mp[3], b.ks, b.M, c.head_dim, c.head_dim, attn::BKEY))) return rc;
    if ((rc = gemm::make_map(&mp[4], b.vt, c.head_dim, b.m_ld, b.m_ld, c.head_dim))) return rc;
  }
  // 2-SM attention for batched rounds (one split): 128-key superblocks, CTA r
  // of a pair loads key block 2G + r and dims [128 r, 128 r + 128) of V^T
  // (default; SF_ATTN_SINGLE=1 selects the 1-SM persistent kernel)
  b.attn_pair = b.attn_splits == 1 && tiles_env >= 2 && getenv("SF_ATTN_SINGLE") == nullptr;
  if (b.attn_pair) {
    b.attn_pair_maps.resize(5 * L);
    for (int l = 0; l < L; ++l) {
      CUtensorMap* mp = &b.attn_pair_maps[5 * l];
      mp[0] = b.attn_maps[5 * l];
      const bf16* kp = h.k_prefix + (size_t)l * E * c.prefix_len * c.head_dim;
      const bf16* vp = h.vt_prefix + (size_t)l * E * c.head_dim * c.prefix_len;
      if ((rc = make_map_3d(&mp[1], kp, c.head_dim, c.prefix_len, E, (uint64_t)c.head_dim * 2,
                            (uint64_t)c.prefix_len * c.head_dim * 2, 64, attn::BKEY)))
        return rc;
      if ((rc = make_map_3d(&mp[2], vp, c.prefix_len, c.head_dim, E, (uint64_t)c.prefix_len * 2,
                            (uint64_t)c.prefix_len * c.head_dim * 2, attn::BKEY, c.head_dim / 2)))
        return rc;
      if ((rc = gemm::make_map(&mp[3], b.ks, b.M, c.head_dim, c.head_dim, attn::BKEY))) return rc;
      if ((rc = gemm::make_map(&mp[4], b.vt, c.head_dim, b.m_ld, b.m_ld, c.head_dim / 2))) return rc;
    }
  }
  return SF_OK;
}

int launch_attn_pair(const Buffers& b, int l, cudaStream_t s, bool pdl) {
  static bool attr = false;
  if (!attr) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(attn::attn_pair_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)attn::kPairSmemBytes));
    attr = true;
  }
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const CUtensorMap* mp = &b.attn_pair_maps[5 * l];
  const int tiles_env = b.ap.tiles_env;
  const int pairs = b.B * ((tiles_env + 1) / 2);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * (pairs < nsm / 2 ? pairs : nsm / 2));  // persistent: one CTA pair per 2 SMs
  cfg.blockDim = dim3(attn::kThreads);
  cfg.dynamicSmemBytes = attn::kPairSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  a[1].id = cudaLaunchAttributeClusterDimension;
  a[1].val.clusterDim.x = 2;
  a[1].val.clusterDim.y = 1;
  a[1].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 2;
  SF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, attn::attn_pair_kernel, mp[0], mp[1], mp[2], mp[3], mp[4], b.ap));
  count_launch();
  return SF_OK;
}

int launch_attn(const Buffers& b, int l, cudaStream_t s, bool pdl) {
  if (b.attn_pair) return launch_attn_pair(b, l, s, pdl);
  if (b.attn_splits == 1 && getenv("SF_NO_ATTN_PERSIST") == nullptr) {
    // batched: persistent CTAs (one per SM) walk the query tiles
    static bool pattr = false;
    static int nsm = 148;
    if (!pattr) {
      SF_CHECK_CUDA(cudaFuncSetAttribute(attn::attn_persistent_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)attn::kPersistSmemBytes));
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      pattr = true;
    }
    const CUtensorMap* mp = &b.attn_maps[5 * l];
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(b.attn_tiles < nsm ? b.attn_tiles : nsm);
    cfg.blockDim = dim3(attn::kThreads);
    cfg.dynamicSmemBytes = attn::kPersistSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    attn::Params ap = b.ap;
    if (b.k_img) {
      const size_t per_layer = (size_t)b.n_img_envs * b.img_blocks * 32768;
      ap.k_img = b.k_img + (size_t)l * per_layer;
      ap.v_img = b.v_img + (size_t)l * per_layer;
      ap.img_blocks = b.img_blocks;
    }
    SF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, attn::attn_persistent_kernel, mp[0], mp[1], mp[2], mp[3], mp[4], ap));
    count_launch();
    return SF_OK;
  }
  static bool attr = false;
  if (!attr) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(attn::attn_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)attn::kSmemBytes));
    SF_CHECK_CUDA(cudaFuncSetAttribute(attn::attn_kernel,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  const CUtensorMap* mp = &b.attn_maps[5 * l];
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(b.attn_tiles, b.attn_splits);
  cfg.blockDim = dim3(attn::kThreads);
  cfg.dynamicSmemBytes = attn::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  int na = 1;
  if (b.attn_splits > 1) {
    a[1].id = cudaLaunchAttributeClusterDimension;
    a[1].val.clusterDim.x = 1;
    a[1].val.clusterDim.y = b.attn_splits;
    a[1].val.clusterDim.z = 1;
    na = 2;
  }
  cfg.attrs = a;
  cfg.numAttrs = na;
  attn::Params ap = b.ap;
  if (b.k_img) {  // this layer's slice of the prefix block images
    const size_t per_layer = (size_t)b.n_img_envs * b.img_blocks * 32768;
    ap.k_img = b.k_img + (size_t)l * per_layer;
    ap.v_img = b.v_img + (size_t)l * per_layer;
    ap.img_blocks = b.img_blocks;
  }
  SF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, attn::attn_kernel, mp[0], mp[1], mp[2], mp[3], mp[4], ap));
  count_launch();
  return SF_OK;
}

// Optional per-kernel event trace (sf_ae_profile_verify): an event is
// recorded after every launch of an eager (non-graph) round.
std::vector<cudaEvent_t>* g_trace = nullptr;
void trace_mark(cudaStream_t s) {
  if (!g_trace) return;
  cudaEvent_t ev;
  cudaEventCreate(&ev);
  cudaEventRecord(ev, s);
  g_trace->push_back(ev);
}

// fp32 mode: the layer stack + head in fp32 on CUDA cores (stack_f32.cuh).
int alloc_f32(Handle& h, Buffers& b) {
  const sf_ae_config_t& c = h.cfg;
  const size_t M = (size_t)b.M, nq = (size_t)c.q_heads * c.head_dim;
  int rc;
  if ((rc = dalloc(&b.f_rs, M)) || (rc = dalloc(&b.f_qkv, M * (nq + 2 * c.head_dim))) ||
      (rc = dalloc(&b.f_q, M * nq)) || (rc = dalloc(&b.f_k, M * c.head_dim)) ||
      (rc = dalloc(&b.f_v, M * c.head_dim)) || (rc = dalloc(&b.f_o, M * nq)) ||
      (rc = dalloc(&b.f_gu, M * 2 * c.mlp)) || (rc = dalloc(&b.f_h, M * c.mlp)))
    return rc;
  b.fp32 = true;
  return SF_OK;
}

int run_stack_f32(Handle& h, Buffers& b, cudaStream_t s) {
  using namespace sf::f32;
  const sf_ae_config_t& c = h.cfg;
  const int M = b.M, W = c.width, nq = c.q_heads * c.head_dim, hd = c.head_dim;
  const int T = T_of(h), L = c.layers, P = c.prefix_len;
  const dim3 rms_grid((M * 32 + 255) / 256);
  auto gemm = [&](bool resid, const float* A, int lda, const void* Wt, int N, int K, const float* rs,
                  const float* bias, float* C, int ldc) {
    const dim3 grid((N + 63) / 64, (M + 63) / 64);
    if (resid)
      gemm_f32_kernel<E_RESID><<<grid, 256, 0, s>>>(A, lda, (const bf16*)Wt, M, N, K, rs, bias, C, ldc);
    else
      gemm_f32_kernel<E_STORE><<<grid, 256, 0, s>>>(A, lda, (const bf16*)Wt, M, N, K, rs, bias, C, ldc);
  };
  const size_t attn_smem = sizeof(float) * ((size_t)NH * 256 + (size_t)NH * (P + T));
  static size_t attn_smem_set = 0;
  if (attn_smem > attn_smem_set) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(attn_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)attn_smem));
    attn_smem_set = attn_smem;
  }
  for (int l = 0; l < L; ++l) {
    rms_rows_kernel<<<rms_grid, 256, 0, s>>>(b.x, M, W, c.eps, b.f_rs);
    gemm(false, b.x, W, h.w.qkv[l], nq + 2 * hd, W, b.f_rs, nullptr, b.f_qkv, nq + 2 * hd);
    RopeParams rp{b.f_qkv, h.rope_t, P + T, M, c.q_heads, b.env_rows, T, P, b.f_q, b.f_k, b.f_v};
    rope_split_f32_kernel<<<M, 256, 0, s>>>(rp);
    AttnParams ap{b.f_q, b.f_k, b.f_v,
                  h.k_prefix + (size_t)l * h.n_prefix_envs * P * hd,
                  h.vt_prefix + (size_t)l * h.n_prefix_envs * hd * P,
                  b.env_map, M, b.B, c.q_heads, b.env_rows, T, b.K, P, 1.f / sqrtf((float)hd), b.f_o};
    attn_f32_kernel<<<M, 256, attn_smem, s>>>(ap);
    gemm(true, b.f_o, nq, h.w.o[l], W, nq, nullptr, nullptr, b.x, W);
    rms_rows_kernel<<<rms_grid, 256, 0, s>>>(b.x, M, W, c.eps, b.f_rs);
    gemm(false, b.x, W, h.w.gu[l], 2 * c.mlp, W, b.f_rs, nullptr, b.f_gu, 2 * c.mlp);
    geglu_f32_kernel<<<592, 256, 0, s>>>(b.f_gu, M, c.mlp, b.f_h);
    gemm(true, b.f_h, c.mlp, h.w.down[l], W, c.mlp, nullptr, nullptr, b.x, W);
  }
  rms_rows_kernel<<<rms_grid, 256, 0, s>>>(b.x, M, W, c.eps, b.f_rs);
  gemm(false, b.x, W, h.w.out_w, c.action_dim, W, b.f_rs, (const float*)h.w.out_b, b.vel, c.action_dim);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch(L * 9 + 2);
  return SF_OK;
}

// The layer stack + head on the current X (used by verify and Euler).
int run_stack(Handle& h, Buffers& b, cudaStream_t s, bool pdl) {
  if (b.fp32) return run_stack_f32(h, b, s);
  int rc;
  for (int l = 0; l < h.cfg.layers; ++l) {
    if ((rc = gemm::launch(b.ops[4 * l + 0], s, pdl))) return rc;
    trace_mark(s);
    if ((rc = launch_attn(b, l, s, pdl))) return rc;
    trace_mark(s);
    if ((rc = gemm::launch(b.ops[4 * l + 1], s, pdl))) return rc;
    trace_mark(s);
    if ((rc = gemm::launch(b.ops[4 * l + 2], s, pdl))) return rc;
    trace_mark(s);
    if ((rc = gemm::launch(b.ops[4 * l + 3], s, pdl))) return rc;
    trace_mark(s);
  }
  rc = gemm::launch(b.ops[4 * h.cfg.layers], s, pdl);
  trace_mark(s);
  return rc;
}

EmbedParams embed_params(const Handle& h, const Buffers& b, int mode, const float* temb) {
  const sf_ae_config_t& c = h.cfg;
  EmbedParams p{};
  p.W = c.width;
  p.D = c.action_dim;
  p.S = c.state_dim;
  p.H = c.horizon;
  p.T = T_of(h);
  p.K = b.K;
  p.env_rows = b.env_rows;
  p.B = b.B;
  p.mode = mode;
  p.draft = b.draft;
  p.eps = b.eps;
  for (int k = 0; k < b.K && k < SF_MAX_K; ++k) p.taus[k] = h.temb_taus[k];
  p.temb = temb;
  p.state = b.state;
  p.a_wt = h.a_wt;
  p.a_b = static_cast<const float*>(h.w.a_b);
  p.s_wt = h.s_wt;
  p.s_b = static_cast<const float*>(h.w.s_b);
  p.x = b.x;
  p.xb = b.xb;
  p.ssq = b.ssq;
  p.ssq_ld = b.m_ld;
  return p;
}

// Verify chain for the staged inputs of `b` (draft/eps/state/signs already in b).
int enqueue_verify(Handle& h, Buffers& b, const sf_verify_cfg_t* cfg, cudaStream_t s, bool pdl,
                   bool with_draft = false) {
  int rc;
  if (with_draft) {
    // propose (draft.py:57-61): obs -> tanh MLP -> draft [B][H][D] into b.draft
    CastParams cp{b.obs, b.obs_b, b.B * h.cfg.draft_in};
    if ((rc = launch_pdl(cast_bf16_kernel, dim3((cp.n + 255) / 256), dim3(256), 0, s, cp, false)))
      return rc;
    for (int i = 0; i < 3; ++i)
      if ((rc = gemm::launch(b.dops[i], s, pdl))) return rc;
  }
  EmbedParams ep = embed_params(h, b, 0, h.temb);
  if ((rc = launch_embed(b.M, h.cfg.width, s, ep, with_draft && pdl))) return rc;
  trace_mark(s);
  if ((rc = run_stack(h, b, s, pdl))) return rc;
  VerifyEpiParams vp{};
  const sf_ae_config_t& c = h.cfg;
  vp.H = c.horizon;
  vp.D = c.action_dim;
  vp.C = c.action_dim - 1;
  vp.K = b.K;
  vp.T = T_of(h);
  vp.env_rows = b.env_rows;
  for (int k = 0; k < b.K; ++k) vp.taus[k] = (float)cfg->taus[k];
  vp.delta = (float)cfg->delta;
  vp.metric = cfg->metric;
  vp.window = cfg->window;
  vp.sign = (float)cfg->current_sign;
  vp.signs = b.signs;
  vp.phase_fallback = cfg->phase_fallback;
  vp.prefix_cap = cfg->prefix_cap;
  vp.replan_size = cfg->replan_size;
  vp.draft = b.draft;
  vp.eps = b.eps;
  vp.vel = b.vel;
  vp.out_recon = b.recon;
  vp.out_dist = b.dist;
  vp.out_branch = b.branch;
  vp.out_result = b.result;
  const size_t smem = sizeof(float) * ((size_t)b.K * c.horizon * c.action_dim + b.K * c.horizon);
  static bool attr = false;
  if (!attr) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(verify_epi_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  rc = launch_pdl(verify_epi_kernel, dim3(b.B), dim3(b.B <= 16 ? 1024 : 256), smem, s, vp, pdl);
  trace_mark(s);
  return rc;
}

int enqueue_denoise(Handle& h, Buffers& b, int n_steps, cudaStream_t s, bool pdl) {
  int rc;
  const int W = h.cfg.width;
  StatusParams sp{b.status, b.B};
  if ((rc = launch_pdl(status_init_kernel, dim3(1), dim3(256), 0, s, sp, false))) return rc;
  for (int i = 0; i < n_steps; ++i) {
    EmbedParams ep = embed_params(h, b, 1, h.temb_euler + (size_t)i * W);
    if ((rc = launch_embed(b.M, h.cfg.width, s, ep, pdl))) return rc;
    if ((rc = run_stack(h, b, s, pdl))) return rc;
    const int total = b.B * h.cfg.horizon * h.cfg.action_dim;
    EulerParams up{b.draft, b.vel, b.B, h.cfg.horizon, h.cfg.action_dim, b.env_rows, n_steps, i,
                   b.status};
    if ((rc = launch_pdl(euler_rows_kernel, dim3((total + 255) / 256), dim3(256), 0, s, up, pdl)))
      return rc;
  }
  return SF_OK;
}

// mode: 0 verify, 1 denoise, 2 velocity; + kModeF32 for the fp32-mode buffers
constexpr int kModeF32 = 8;
Buffers* get_buffers(Handle& h, int B, int K, int mode, int* rc) {
  const long long key = ((long long)mode << 40) | ((long long)B << 8) | K;
  auto it = h.buffers.find(key);
  if (it != h.buffers.end()) return it->second.get();
  auto b = std::make_unique<Buffers>();
  *rc = build(h, *b, B, K);
  if (*rc) return nullptr;
  if ((mode & kModeF32) && (*rc = alloc_f32(h, *b))) return nullptr;
  Buffers* raw = b.get();
  h.buffers[key] = std::move(b);
  return raw;
}

// Capture `fn(stream)` into a graph on the handle's capture stream.
template <typename F>
int capture(Handle& h, cudaGraphExec_t* exec, int* n_kernels, F&& fn) {
  if (!h.capture_stream)
    SF_CHECK_CUDA(cudaStreamCreateWithFlags(&h.capture_stream, cudaStreamNonBlocking));
  cudaGraph_t g = nullptr;
  SF_CHECK_CUDA(cudaStreamBeginCapture(h.capture_stream, cudaStreamCaptureModeThreadLocal));
  const int64_t before = sf_launch_count(0);
  const int rc = fn(h.capture_stream);
  // captured kernels are recorded, not launched: they count on each replay
  *n_kernels = (int)(sf_launch_count(0) - before);
  count_launch(-*n_kernels);
  cudaError_t e = cudaStreamEndCapture(h.capture_stream, &g);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  SF_CHECK_CUDA(e);
  if (*exec) cudaGraphExecDestroy(*exec);
  e = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  SF_CHECK_CUDA(e);
  return SF_OK;
}

int cfg_key(const sf_verify_cfg_t* c) {
  // cheap hash of the verify knobs baked into the graph's kernel params
  uint64_t hsh = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) hsh = (hsh ^ b[i]) * 1099511628211ull;
  };
  mix(c, sizeof(*c));
  return (int)(hsh & 0x7fffffff);
}

}  // namespace pi0
}  // namespace sf

using namespace sf::pi0;

extern "C" int sf_fill_hash_uniform(void* dst, int is_bf16, int64_t n, uint64_t seed, uint64_t tid,
                                    double std_, void* stream) {
  SF_REQUIRE(dst && n >= 0, "bad fill arguments");
  if (n == 0) return SF_OK;
  const float a = (float)(std_ * 1.7320508075688772);  // np.float32(std * np.sqrt(3.0))
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  fill_hash_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(dst, is_bf16, n, seed, tid, a);
  SF_CHECK_CUDA(cudaGetLastError());
  sf::count_launch();
  return SF_OK;
}

extern "C" int sf_ae_create(const sf_ae_config_t* cfg, const sf_ae_weights_t* w, void** handle) {
  SF_REQUIRE(cfg && w && handle, "null argument");
  SF_REQUIRE(cfg->head_dim == 256, "head_dim must be 256");
  SF_REQUIRE(cfg->q_heads == 8, "the attention kernel is built for 8 query heads");
  SF_REQUIRE(cfg->width % 256 == 0 && cfg->width <= 2048, "width must be a multiple of 256");
  SF_REQUIRE(cfg->layers >= 1 && cfg->layers <= SF_AE_MAX_LAYERS, "bad layer count");
  SF_REQUIRE(cfg->mlp % 64 == 0, "mlp must be a multiple of 64");
  SF_REQUIRE(cfg->action_dim >= 2 && cfg->action_dim <= 64, "action_dim must be in [2, 64]");
  SF_REQUIRE(cfg->state_dim >= 1 && cfg->state_dim <= 64, "state_dim must be in [1, 64]");
  SF_REQUIRE(cfg->horizon >= 1 && cfg->prefix_len >= 1, "bad horizon / prefix");
  SF_REQUIRE(cfg->draft_in == 0 || (cfg->draft_in % 64 == 0 && cfg->draft_hidden >= 64 &&
                                    cfg->draft_hidden % 64 == 0 && w->draft_w[0] &&
                                    w->draft_w[1] && w->draft_w[2]),
             "draft dims must be multiples of 64 with all three layers given");
  auto* h = new Handle();
  h->cfg = *cfg;
  h->w = *w;
  int rc;
  if ((rc = dalloc(&h->temb, (size_t)SF_MAX_K * cfg->width)) ||
      (rc = dalloc(&h->temb_hidden, (size_t)64 * cfg->width)) ||
      (rc = dalloc(&h->temb_tau_dev, 64)) ||
      (rc = dalloc(&h->a_wt, (size_t)cfg->action_dim * cfg->width)) ||
      (rc = dalloc(&h->s_wt, (size_t)cfg->state_dim * cfg->width)) ||
      (rc = dalloc(&h->rope_t, (size_t)(cfg->head_dim / 2) * (cfg->prefix_len + 1 + cfg->horizon)))) {
    delete h;
    return rc;
  }
  // the embedding weights are read transposed (coalesced); the weights are
  // immutable for the handle's lifetime (sf_ae_create contract)
  transpose_f32_kernel<<<64, 256>>>(static_cast<const float*>(w->a_w), h->a_wt, cfg->width,
                                    cfg->action_dim);
  transpose_f32_kernel<<<64, 256>>>(static_cast<const float*>(w->s_w), h->s_wt, cfg->width,
                                    cfg->state_dim);
  transpose_u64_kernel<<<64, 256>>>(static_cast<const unsigned long long*>(w->rope),
                                    reinterpret_cast<unsigned long long*>(h->rope_t),
                                    cfg->prefix_len + 1 + cfg->horizon, cfg->head_dim / 2);
  SF_CHECK_CUDA(cudaGetLastError());
  SF_CHECK_CUDA(cudaDeviceSynchronize());
  *handle = h;
  return SF_OK;
}

// Drop every plan / graph / activation buffer (they bake the prefix pool's
// tensor maps and pointers); the replanning graphs go first (they reference
// the buffers).
static void free_buffers(Handle* h) {
  h->replans.clear();
  for (auto& kv : h->buffers) {
    Buffers& b = *kv.second;
    if (b.graph) cudaGraphExecDestroy(b.graph);
    void* ptrs[] = {b.x, b.xb, b.ssq, b.q, b.ks, b.vt, b.attn, b.h, b.vel, b.draft, b.eps,
                    b.state, b.signs, b.recon, b.dist, b.branch, b.result, b.status, b.ws,
                    b.counters, b.ap.ws, b.env_map, b.env_ident,
                    b.obs, b.obs_b, b.dh1, b.dh2, b.f_rs, b.f_qkv, b.f_q, b.f_k, b.f_v, b.f_o,
                    b.f_gu, b.f_h};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
  h->buffers.clear();
}

namespace sf {
namespace pi0 {
// ----------------------------------------------------------- batch-1 engine
// The persistent one-launch Euler full path (b1engine.cuh) for n_envs == 1:
// device buffers + weight tensor maps, built on first use.
struct B1Engine {
  b1::Params p{};
  float *x = nullptr, *acc_qkv = nullptr, *acc_gu = nullptr, *acc_head = nullptr, *ssq = nullptr, *A = nullptr;
  bf16 *part_o = nullptr, *qb = nullptr, *kb = nullptr, *vt = nullptr, *xb = nullptr, *hb = nullptr;
  unsigned* cnt = nullptr;
  size_t ssq_n = 0;
  float2* part_ml = nullptr;
  unsigned* bar = nullptr;
  unsigned long long* dbg = nullptr;
  size_t dbg_n = 0;
};

static void destroy_b1(Handle* h) {
  if (!h->b1) return;
  B1Engine& e = *h->b1;
  void* ptrs[] = {e.x, e.acc_qkv, e.acc_gu, e.acc_head, e.ssq, e.A, e.part_o, e.part_ml, e.bar, e.dbg,
                  e.qb, e.kb, e.vt, e.xb, e.hb, e.cnt};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  delete h->b1;
  h->b1 = nullptr;
}

// The engine's static plan is written for the pi0-scale geometry (width 1024,
// 8 x 256 heads, GeGLU 4096, <= 64 suffix tokens) on a 148-SM part.
static bool b1_supported(const Handle& h) {
  const sf_ae_config_t& c = h.cfg;
  if (getenv("SF_NO_B1ENGINE")) return false;
  if (c.width != b1::kW || c.q_heads != b1::kHeads || c.head_dim != b1::kHD || c.mlp != b1::kMlp) return false;
  if (c.horizon + 1 > b1::kTok || c.action_dim % 4 != 0 || c.action_dim > 32 || c.layers > b1::kMaxL) return false;
  if (c.state_dim > 256) return false;  // the E stage stages 8 state-weight rows + the state in 16 KB
  if (!h.k_img || c.prefix_len < 64) return false;
  static int nsm = -1;
  if (nsm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm >= b1::kGrid;
}

static int build_b1(Handle& h) {
  if (h.b1) return SF_OK;
  const sf_ae_config_t& c = h.cfg;
  auto e = std::make_unique<B1Engine>();
  int rc;
  const int L = c.layers, T = 1 + c.horizon;
  if ((rc = dalloc(&e->x, (size_t)b1::kTok * b1::kW)) || (rc = dalloc(&e->acc_qkv, (size_t)b1::kTok * b1::kQKV)) ||
      (rc = dalloc(&e->acc_gu, (size_t)b1::kTok * 2 * b1::kMlp)) ||
      (rc = dalloc(&e->acc_head, (size_t)b1::kTok * c.action_dim)) ||
      (rc = dalloc(&e->ssq, (size_t)(2 * L + 1) * b1::kTok)) ||
      (rc = dalloc(&e->xb, (size_t)b1::kTok * b1::kW)) || (rc = dalloc(&e->hb, (size_t)b1::kTok * b1::kMlp)) ||
      (rc = dalloc(&e->cnt, (size_t)8 * 64)) ||
      (rc = dalloc(&e->A, (size_t)2 * c.horizon * c.action_dim)) ||
      (rc = dalloc(&e->part_o, (size_t)b1::kAttQT * b1::kAttSplits * 128 * b1::kHD)) ||
      (rc = dalloc(&e->part_ml, (size_t)b1::kAttQT * b1::kAttSplits * 128)) || (rc = dalloc(&e->bar, 64)) ||
      (rc = dalloc(&e->qb, (size_t)b1::kTok * b1::kQF)) || (rc = dalloc(&e->kb, (size_t)b1::kTok * b1::kHD)) ||
      (rc = dalloc(&e->vt, (size_t)b1::kHD * b1::kTok)))
    return rc;
  b1::Params& p = e->p;
  for (int l = 0; l < L; ++l) {
    if ((rc = gemm::make_map(&p.wmap[4 * l + 0], h.w.qkv[l], b1::kQKV, b1::kW, b1::kW, 128)) ||
        (rc = gemm::make_map(&p.wmap[4 * l + 1], h.w.o[l], b1::kW, b1::kQF, b1::kQF, 128)) ||
        (rc = gemm::make_map(&p.wmap[4 * l + 2], h.w.gu[l], 2 * b1::kMlp, b1::kW, b1::kW, 128)) ||
        (rc = gemm::make_map(&p.wmap[4 * l + 3], h.w.down[l], b1::kW, b1::kMlp, b1::kMlp, 128)) ||
        (rc = gemm::make_map(&p.wmap64[2 * l + 0], h.w.qkv[l], b1::kQKV, b1::kW, b1::kW, 64)) ||
        (rc = gemm::make_map(&p.wmap64[2 * l + 1], h.w.gu[l], 2 * b1::kMlp, b1::kW, b1::kW, 64)))
      return rc;
  }
  if ((rc = gemm::make_map(&p.wmap[4 * L], h.w.out_w, c.action_dim, b1::kW, b1::kW, 128)) ||
      (rc = gemm::make_map(&p.qmap, e->qb, b1::kTok * b1::kHeads, b1::kHD, b1::kHD, 128)) ||
      (rc = gemm::make_map(&p.kmap, e->kb, b1::kTok, b1::kHD, b1::kHD, 64)) ||
      (rc = gemm::make_map(&p.vmap, e->vt, b1::kHD, b1::kTok, b1::kTok, 256)) ||
      (rc = gemm::make_map(&p.xmap, e->xb, b1::kTok, b1::kW, b1::kW, 64)) ||
      (rc = gemm::make_map(&p.hmap, e->hb, b1::kTok, b1::kMlp, b1::kMlp, 64)) ||
      (rc = gemm::make_map(&p.pmap, e->part_o, b1::kAttQT * b1::kAttSplits * 128, b1::kHD, b1::kHD, 128)))
    return rc;
  e->ssq_n = (size_t)(2 * L + 1) * b1::kTok;
  p.xb = e->xb;
  p.hb = e->hb;
  p.cnt = e->cnt;
  p.qb = e->qb;
  p.kb = e->kb;
  p.vt = e->vt;
  p.L = L;
  p.T = T;
  p.H = c.horizon;
  p.D = c.action_dim;
  p.S = c.state_dim;
  p.P = c.prefix_len;
  p.npb = (c.prefix_len + 63) / 64;
  // KV splits over npb prefix blocks + 1 suffix block; the last split holds
  // the suffix block and at most one prefix block (its worker-written ring
  // items must fit the 4-slot ring at the task start)
  {
    const int nbk = p.npb + 1;
    const int last = p.npb >= 1 ? 2 : 1;
    const int rest = nbk - last, per = (rest + b1::kAttSplits - 2) / (b1::kAttSplits - 1);
    p.att_b[0] = 0;
    for (int s = 1; s < b1::kAttSplits; ++s) p.att_b[s] = std::min(rest, p.att_b[s - 1] + per);
    p.att_b[b1::kAttSplits] = nbk;
  }
  p.inv_width = 1.f / (float)c.width;
  p.eps = c.eps;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)c.head_dim);
  p.rope = static_cast<const float2*>(h.w.rope);
  p.a_w = static_cast<const float*>(h.w.a_w);
  p.a_b = static_cast<const float*>(h.w.a_b);
  p.s_w = static_cast<const float*>(h.w.s_w);
  p.s_b = static_cast<const float*>(h.w.s_b);
  p.out_b = static_cast<const float*>(h.w.out_b);
  p.x = e->x;
  p.acc_qkv = e->acc_qkv;
  p.acc_gu = e->acc_gu;
  p.acc_head = e->acc_head;
  p.ssq1 = e->ssq;                                // [L + 1][64]
  p.ssq2 = e->ssq + (size_t)(L + 1) * b1::kTok;   // [L][64]
  p.A = e->A;
  p.part_o = e->part_o;
  p.part_ml = e->part_ml;
  p.bar = e->bar;
  SF_CHECK_CUDA(cudaFuncSetAttribute(b1::engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)b1::kSmemBytes));
  h.b1 = e.release();
  return SF_OK;
}

// One Euler full round of one env (flowpolicy.py:273-292) as one cooperative
// launch: start/state/chunk_out/status are device pointers (sf_ae_denoise).
static int run_b1(Handle& h, int num_steps, const float* start, const float* state, const int* env_map,
                  float* chunk_out, int* status, cudaStream_t s) {
  int rc;
  if ((rc = build_b1(h))) return rc;
  B1Engine& e = *h.b1;
  const sf_ae_config_t& c = h.cfg;
  b1::Params p = e.p;
  p.n_steps = num_steps;
  p.temb = h.temb_euler;
  p.state = state;
  p.env_map = env_map;
  p.k_img = h.k_img;
  p.v_img = h.v_img;
  p.n_img_envs = h.n_prefix_envs;
  p.chunk_out = chunk_out;
  p.status = status;
  const int n_st = b1::stages_per_step(p.L) * num_steps + 1;
  if (getenv("SF_B1_TRACE")) {
    const size_t n = (size_t)b1::kGrid * n_st * 8;
    if (e.dbg_n < n) {
      if (e.dbg) cudaFree(e.dbg);
      e.dbg = nullptr;
      if ((rc = dalloc(&e.dbg, n))) return rc;
      e.dbg_n = n;
    }
    p.dbg = e.dbg;
  }
  SF_CHECK_CUDA(cudaMemsetAsync(e.bar, 0, 64, s));
  SF_CHECK_CUDA(cudaMemsetAsync(e.cnt, 0, sizeof(unsigned) * 8 * 64, s));
  SF_CHECK_CUDA(cudaMemsetAsync(e.ssq, 0, sizeof(float) * e.ssq_n, s));
  SF_CHECK_CUDA(cudaMemcpyAsync(e.A, start, sizeof(float) * c.horizon * c.action_dim, cudaMemcpyDeviceToDevice, s));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(b1::kGrid);
  cfg.blockDim = dim3(b1::kThreads);
  cfg.dynamicSmemBytes = b1::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeCooperative;
  a[0].val.cooperative = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  SF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, b1::engine_kernel, p));
  count_launch();
  return SF_OK;
}
}  // namespace pi0
}  // namespace sf

extern "C" int sf_ae_b1_trace(void* handle, unsigned long long* out, size_t n) {
  auto* h = static_cast<Handle*>(handle);
  SF_REQUIRE(h && out, "null argument");
  SF_REQUIRE(h->b1 && h->b1->dbg && n <= h->b1->dbg_n, "no batch-1 engine trace (run with SF_B1_TRACE=1)");
  SF_CHECK_CUDA(cudaDeviceSynchronize());
  SF_CHECK_CUDA(cudaMemcpy(out, h->b1->dbg, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return SF_OK;
}

extern "C" int sf_ae_destroy(void* handle) {
  auto* h = static_cast<Handle*>(handle);
  if (!h) return SF_OK;
  free_buffers(h);
  cudaFree(h->temb);
  cudaFree(h->temb_hidden);
  cudaFree(h->temb_tau_dev);
  cudaFree(h->a_wt);
  cudaFree(h->s_wt);
  cudaFree(h->rope_t);
  if (h->k_img) cudaFree(h->k_img);
  if (h->v_img) cudaFree(h->v_img);
  if (h->temb_euler) cudaFree(h->temb_euler);
  if (h->capture_stream) cudaStreamDestroy(h->capture_stream);
  if (h->body_stream) cudaStreamDestroy(h->body_stream);
  destroy_b1(h);
  delete h;
  return SF_OK;
}

extern "C" int sf_ae_set_prefix(void* handle, const void* k_prefix, const void* vt_prefix,
                                int n_envs) {
  auto* h = static_cast<Handle*>(handle);
  SF_REQUIRE(h && k_prefix && vt_prefix && n_envs >= 1, "bad prefix arguments");
  h->k_prefix = static_cast<const bf16*>(k_prefix);
  h->vt_prefix = static_cast<const bf16*>(vt_prefix);
  h->n_prefix_envs = n_envs;
  // block images of the pool (re-laid out once; the attention streams each
  // 64-key block of K and V^T with one bulk copy)
  {
    const sf_ae_config_t& c = h->cfg;
    if (h->k_img) cudaFree(h->k_img);
    if (h->v_img) cudaFree(h->v_img);
    h->k_img = h->v_img = nullptr;
    h->img_blocks = 0;
    const int nblk = (c.prefix_len + 63) / 64;
    const size_t bytes = (size_t)c.layers * n_envs * nblk * 32768;
    if (getenv("SF_NO_KV_IMAGES") == nullptr && c.head_dim == 256 &&
        cudaMalloc(&h->k_img, bytes) == cudaSuccess && cudaMalloc(&h->v_img, bytes) == cudaSuccess) {
      // the pool may have been written on any stream (setup call: full sync)
      SF_CHECK_CUDA(cudaDeviceSynchronize());
      prefix_image_kernel<<<148 * 8, 256>>>(h->k_prefix, h->vt_prefix, h->k_img, h->v_img,
                                            c.layers * n_envs, c.prefix_len, nblk);
      SF_CHECK_CUDA(cudaGetLastError());
      SF_CHECK_CUDA(cudaDeviceSynchronize());
      h->img_blocks = nblk;
    } else {
      cudaGetLastError();  // out of memory is not fatal: the tensor-map path stays
      if (h->k_img) cudaFree(h->k_img);
      h->k_img = nullptr;
    }
  }
  // plans embed the prefix tensor maps: drop them
  free_buffers(h);
  return SF_OK;
}

// Re-derive the attention's block images after the bound pool was rewritten
// in place (a context refresh, e.g. sf_vlm_prefill into the bound pool), on
// `stream` after that write. Graphs stay valid (same image pointers).
extern "C" int sf_ae_refresh_prefix(void* handle, void* stream) {
  auto* h = static_cast<Handle*>(handle);
  SF_REQUIRE(h && h->k_prefix, "no prefix KV bound (sf_ae_set_prefix)");
  if (!h->k_img) return SF_OK;  // tensor-map path reads the pool directly
  const sf_ae_config_t& c = h->cfg;
  prefix_image_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
      h->k_prefix, h->vt_prefix, h->k_img, h->v_img, c.layers * h->n_prefix_envs, c.prefix_len, h->img_blocks);
  SF_CHECK_CUDA(cudaGetLastError());
  sf::count_launch();
  return SF_OK;
}

static int ensure_temb(Handle& h, const sf_verify_cfg_t* cfg, cudaStream_t s) {
  bool same = h.temb_k == cfg->k;
  for (int k = 0; same && k < cfg->k; ++k) same = h.temb_taus[k] == (float)cfg->taus[k];
  if (same) return SF_OK;
  for (int k = 0; k < cfg->k; ++k) h.temb_taus[k] = (float)cfg->taus[k];
  h.temb_k = cfg->k;
  return compute_temb(h, h.temb_taus, cfg->k, h.temb, s);
}

static int check_verify_cfg(const sf_verify_cfg_t* cfg, const float* signs) {
  SF_REQUIRE(cfg->k >= 1 && cfg->k <= SF_MAX_K, "need 1..%d verification timesteps", SF_MAX_K);
  for (int i = 0; i < cfg->k; ++i) {
    SF_REQUIRE(cfg->taus[i] > 0.0 && cfg->taus[i] < 1.0,
               "verification timesteps must lie strictly inside (0, 1)");
    if (i) SF_REQUIRE(cfg->taus[i] > cfg->taus[i - 1], "verification timesteps must be strictly increasing");
  }
  SF_REQUIRE(cfg->delta >= 0.0, "delta must be non-negative");
  SF_REQUIRE(cfg->metric == SF_METRIC_L2 || cfg->metric == SF_METRIC_LINF, "unknown metric");
  SF_REQUIRE(signs || cfg->current_sign == 1.0 || cfg->current_sign == -1.0,
             "current_sign must be -1.0 or +1.0");
  SF_REQUIRE(cfg->replan_size >= 1, "replan_size must be >= 1");
  return SF_OK;
}

// Shared body of sf_ae_verify / sf_ae_flash_round. `in` is the draft
// [B][H][D] (with_draft = false) or the draft features [B][F] (true).
static int verify_common(Handle* h, int n_envs, const sf_verify_cfg_t* cfg, const float* in,
                         bool with_draft, const float* eps, const float* state, const float* signs,
                         const sf_verify_out_t* out, int flags, cudaStream_t s) {
  SF_REQUIRE(h && cfg && in && eps && state && out && out->branch_prefixes && out->result,
             "null argument");
  SF_REQUIRE(h->k_prefix, "no prefix KV bound (sf_ae_set_prefix)");
  SF_REQUIRE(n_envs >= 1 && n_envs <= h->n_prefix_envs, "n_envs exceeds the prefix pool");
  int rc = check_verify_cfg(cfg, signs);
  if (rc) return rc;
  Buffers* b = get_buffers(*h, n_envs, cfg->k, (flags & SF_AE_FP32) ? kModeF32 : 0, &rc);
  if (!b) return rc;
  SF_REQUIRE(!with_draft || b->has_draft, "this expert was built without a draft model");
  if ((rc = ensure_temb(*h, cfg, s))) return rc;
  const sf_ae_config_t& c = h->cfg;
  const size_t hd = (size_t)n_envs * c.horizon * c.action_dim;
  // inputs -> the graph's buffers in one launch (a missing signs vector is
  // one sign for every env, filled on the stream: no host staging, no sync)
  CopyList cin{};
  if (with_draft)
    copy_list_add(cin, b->obs, in, (long long)n_envs * c.draft_in);
  else
    copy_list_add(cin, b->draft, in, (long long)hd);
  copy_list_add(cin, b->eps, eps, (long long)hd);
  copy_list_add(cin, b->state, state, (long long)n_envs * c.state_dim);
  copy_list_add(cin, b->signs, signs, n_envs, (float)cfg->current_sign);
  if ((rc = copy_list_launch(cin, s))) return rc;
  const bool pdl = (flags & SF_AE_PDL) != 0;
  if (flags & SF_AE_GRAPH) {
    const int key = cfg_key(cfg) ^ (pdl ? 0x5bd1e995 : 0) ^ (with_draft ? 0x2f3a7c11 : 0);
    if (!b->graph || b->graph_key != key) {
      rc = capture(*h, &b->graph, &b->graph_kernels, [&](cudaStream_t cs) {
        return enqueue_verify(*h, *b, cfg, cs, pdl, with_draft);
      });
      if (rc) return rc;
      b->graph_key = key;
    }
    SF_CHECK_CUDA(cudaGraphLaunch(b->graph, s));
    sf::count_launch(b->graph_kernels);
  } else {
    if ((rc = enqueue_verify(*h, *b, cfg, s, pdl, with_draft))) return rc;
  }
  const size_t khd = hd * cfg->k;
  CopyList co{};
  if (out->draft) copy_list_add(co, out->draft, b->draft, (long long)hd);
  if (out->reconstructed) copy_list_add(co, out->reconstructed, b->recon, (long long)khd);
  if (out->distances) copy_list_add(co, out->distances, b->dist, (long long)n_envs * cfg->k * c.horizon);
  copy_list_add(co, out->branch_prefixes, b->branch, (long long)n_envs * cfg->k);
  copy_list_add(co, out->result, b->result, (long long)n_envs * SF_RESULT_WORDS);
  return copy_list_launch(co, s);
}

extern "C" int sf_ae_verify(void* handle, int n_envs, const sf_verify_cfg_t* cfg, const float* draft,
                            const float* eps, const float* state, const float* signs,
                            const sf_verify_out_t* out, int flags, void* stream) {
  return verify_common(static_cast<Handle*>(handle), n_envs, cfg, draft, false, eps, state, signs,
                       out, flags, (cudaStream_t)stream);
}

extern "C" int sf_ae_flash_round(void* handle, int n_envs, const sf_verify_cfg_t* cfg,
                                 const float* obs, const float* eps, const float* state,
                                 const float* signs, const sf_verify_out_t* out, int flags,
                                 void* stream) {
  return verify_common(static_cast<Handle*>(handle), n_envs, cfg, obs, true, eps, state, signs,
                       out, flags, (cudaStream_t)stream);
}

extern "C" int sf_ae_time_op(void* handle, int n_envs, int k, int op, int iters, void* stream) {
  auto* h = static_cast<Handle*>(handle);
  SF_REQUIRE(h && h->k_prefix, "no expert / prefix");
  int rc = 0;
  Buffers* b = get_buffers(*h, n_envs, k, 0, &rc);
  if (!b) return rc;
  SF_REQUIRE(op >= 0 && op < (int)b->ops.size(), "op index out of range");
  for (int i = 0; i < iters; ++i)
    if ((rc = sf::gemm::launch(b->ops[op], (cudaStream_t)stream, false))) return rc;
  return SF_OK;
}

// Per-kernel warm timings of one eager verify round (no graph, no PDL):
// times_us[i] = device time between consecutive launches, in launch order
// (embed, 18 x [qkv, attn, o, gate/up, down], head, epilogue).
extern "C" int sf_ae_profile_verify(void* handle, int n_envs, const sf_verify_cfg_t* cfg,
                                    const float* draft, const float* eps, const float* state,
                                    float* times_us, int max_times, int* n_times, void* stream) {
  auto* h = static_cast<Handle*>(handle);
  SF_REQUIRE(h && cfg && draft && eps && state && times_us && n_times, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = check_verify_cfg(cfg, nullptr);
  if (rc) return rc;
  Buffers* b = get_buffers(*h, n_envs, cfg->k, 0, &rc);
  if (!b) return rc;
  if ((rc = ensure_temb(*h, cfg, s))) return rc;
  const sf_ae_config_t& c = h->cfg;
  const size_t hd = (size_t)n_envs * c.horizon * c.action_dim;
  SF_CHECK_CUDA(cudaMemcpyAsync(b->draft, draft, hd * 4, cudaMemcpyDeviceToDevice, s));
  SF_CHECK_CUDA(cudaMemcpyAsync(b->eps, eps, hd * 4, cudaMemcpyDeviceToDevice, s));
  SF_CHECK_CUDA(cudaMemcpyAsync(b->state, state, (size_t)n_envs * c.state_dim * 4,
                                cudaMemcpyDeviceToDevice, s));
  std::vector<cudaEvent_t> evs;
  // hold the stream while the host enqueues, so the trace measures the GPU
  SleepParams sp{3000000};
  if ((rc = launch_pdl(sleep_kernel, dim3(1), dim3(32), 0, s, sp, false))) return rc;
  g_trace = &evs;
  trace_mark(s);
  rc = enqueue_verify(*h, *b, cfg, s, false, false);
  g_trace = nullptr;
  SF_CHECK_CUDA(cudaStreamSynchronize(s));
  int n = 0;
  for (size_t i = 1; i < evs.size() && n < max_times; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, evs[i - 1], evs[i]);
    times_us[n++] = ms * 1e3f;
  }
  for (auto ev : evs) cudaEventDestroy(ev);
  *n_times = n;
  return rc;
}

extern "C" int sf_ae_denoise_envs(void* handle, int n_envs, const int* env_map, int num_steps,
                                  const float* start, const float* state, float* chunk_out,
                                  int* status, int flags, void* stream);

// Euler time embeddings for tau_i = i / N; every captured denoise graph and
// replanning graph baked the previous table's pointer, so all are dropped.
static int set_euler_steps(Handle& h, int num_steps, cudaStream_t s) {
  if (h.temb_euler_n == num_steps) return SF_OK;
  int rc;
  h.replans.clear();
  for (auto& kv : h.buffers)
    if (kv.second->graph && kv.second->graph_key & 0x40000000) {
      cudaGraphExecDestroy(kv.second->graph);
      kv.second->graph = nullptr;
    }
  if (h.temb_euler) cudaFree(h.temb_euler);
  h.temb_euler = nullptr;
  if ((rc = dalloc(&h.temb_euler, (size_t)num_steps * h.cfg.width))) return rc;
  std::vector<float> taus(num_steps);
  for (int i = 0; i < num_steps; ++i) taus[i] = (float)((double)i / (double)num_steps);
  if ((rc = compute_temb(h, taus.data(), num_steps, h.temb_euler, s))) return rc;
  SF_CHECK_CUDA(cudaStreamSynchronize(s));
  h.temb_euler_n = num_steps;
  return SF_OK;
}

extern "C" int sf_ae_denoise(void* handle, int n_envs, int num_steps, const float* start,
                             const float* state, float* chunk_out, int* status, int flags,
                             void* stream) {
  return sf_ae_denoise_envs(handle, n_envs, nullptr, num_steps, start, state, chunk_out, status,
                            flags, stream);
}

extern "C" int sf_ae_denoise_envs(void* handle, int n_envs, const int* env_map, int num_steps,
                                  const float* start, const float* state, float* chunk_out,
                                  int* status, int flags, void* stream) {
  auto* h = static_cast<Handle*>(handle);
  SF_REQUIRE(h && start && state && chunk_out && status, "null argument");
  SF_REQUIRE(h->k_prefix, "no prefix KV bound (sf_ae_set_prefix)");
  SF_REQUIRE(n_envs >= 1 && n_envs <= h->n_prefix_envs, "n_envs exceeds the prefix pool");
  SF_REQUIRE(num_steps >= 1 && num_steps <= 64, "num_steps must be in [1, 64]");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = 0;
  if (n_envs == 1 && !(flags & SF_AE_FP32) && b1_supported(*h)) {
    // batch 1: the whole round is one persistent launch (b1engine.cuh)
    if ((rc = set_euler_steps(*h, num_steps, s))) return rc;
    return run_b1(*h, num_steps, start, state, env_map, chunk_out, status, s);
  }
  Buffers* b = get_buffers(*h, n_envs, 1, 1 | ((flags & SF_AE_FP32) ? kModeF32 : 0), &rc);
  if (!b) return rc;
  const sf_ae_config_t& c = h->cfg;
  if ((rc = set_euler_steps(*h, num_steps, s))) return rc;
  const size_t hd = (size_t)n_envs * c.horizon * c.action_dim;
  // batch env e attends to pool slot env_map[e] (fallback envs compacted by
  // sf_replan_update); identity when no map is given
  CopyList cin{};
  copy_list_add(cin, b->env_map, env_map ? env_map : b->env_ident, n_envs);
  copy_list_add(cin, b->draft, start, (long long)hd);
  copy_list_add(cin, b->state, state, (long long)n_envs * c.state_dim);
  if ((rc = copy_list_launch(cin, s))) return rc;
  const bool pdl = (flags & SF_AE_PDL) != 0;
  if (flags & SF_AE_GRAPH) {
    const int key = 0x40000000 | (num_steps << 1) | (pdl ? 1 : 0);
    if (!b->graph || b->graph_key != key) {
      rc = capture(*h, &b->graph, &b->graph_kernels, [&](cudaStream_t cs) {
        return enqueue_denoise(*h, *b, num_steps, cs, pdl);
      });
      if (rc) return rc;
      b->graph_key = key;
    }
    SF_CHECK_CUDA(cudaGraphLaunch(b->graph, s));
    sf::count_launch(b->graph_kernels);
  } else {
    if ((rc = enqueue_denoise(*h, *b, num_steps, s, pdl))) return rc;
  }
  CopyList co{};
  copy_list_add(co, chunk_out, b->draft, (long long)hd);
  copy_list_add(co, status, b->status, 2LL * n_envs);
  return copy_list_launch(co, s);
}

namespace {

// Euler buckets: powers of two up to 64, then multiples of 64, capped at n
std::vector<int> replan_buckets(int n) {
  std::vector<int> b;
  for (int v = 1; v < 64 && v < n; v *= 2) b.push_back(v);
  for (int v = 64; v < n; v += 64) b.push_back(v);
  b.push_back(n);
  return b;
}

// flash-attempt buckets: powers of two up to 32, then multiples of 32, capped
// at n (the attempt costs ~4x an Euler step per env: finer steps)
std::vector<int> flash_buckets(int n) {
  std::vector<int> b;
  for (int v = 1; v < 32 && v < n; v *= 2) b.push_back(v);
  for (int v = 32; v < n; v += 32) b.push_back(v);
  b.push_back(n);
  return b;
}

// conditional handle of a SWITCH over `nb` bodies in the graph being captured on cs
int make_switch_handle(cudaStream_t cs, int nb, cudaGraphConditionalHandle* cond) {
  cudaStreamCaptureStatus st;
  cudaGraph_t cg = nullptr;
  if (cudaStreamGetCaptureInfo(cs, &st, nullptr, &cg, nullptr, nullptr) != cudaSuccess || !cg) return SF_ECUDA;
  if (cudaGraphConditionalHandleCreate(cond, cg, (unsigned)nb, cudaGraphCondAssignDefault) != cudaSuccess) {
    sf::set_error("cudaGraphConditionalHandleCreate failed");
    return SF_ECUDA;
  }
  return SF_OK;
}

// the SWITCH node at the capture position of cs (its bodies: cp->conditional.phGraph_out)
int add_switch_node(cudaStream_t cs, cudaGraphConditionalHandle cond, int nb, cudaGraphNodeParams* cp) {
  cudaStreamCaptureStatus st;
  cudaGraph_t cg = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  if (cudaStreamGetCaptureInfo(cs, &st, nullptr, &cg, &deps, &ndeps) != cudaSuccess) return SF_ECUDA;
  memset(cp, 0, sizeof(*cp));
  cp->type = cudaGraphNodeTypeConditional;
  cp->conditional.handle = cond;
  cp->conditional.type = cudaGraphCondTypeSwitch;
  cp->conditional.size = (unsigned)nb;
  cudaGraphNode_t node;
  const cudaError_t ce = cudaGraphAddNode(&node, cg, deps, ndeps, cp);
  if (ce != cudaSuccess) {
    sf::set_error("conditional SWITCH node: %s", cudaGetErrorString(ce));
    return SF_ECUDA;
  }
  if (cudaStreamUpdateCaptureDependencies(cs, &node, 1, cudaStreamSetCaptureDependencies) != cudaSuccess)
    return SF_ECUDA;
  return SF_OK;
}

int build_replan(Handle& h, Replan& R, int n, const sf_verify_cfg_t* cfg, const sf_replan_policy_t* pol,
                 const float* signs_unused, int* fsr, int* has_cache, bool pdl, bool fp32) {
  (void)signs_unused;
  const sf_ae_config_t& c = h.cfg;
  const int hd = c.horizon * c.action_dim;
  int rc = 0;
  R.n = n;
  R.K = cfg->k;
  const int f32mode = fp32 ? kModeF32 : 0;
  R.bf = get_buffers(h, n, cfg->k, f32mode, &rc);
  if (!R.bf) return rc;
  SF_REQUIRE(R.bf->has_draft, "the replanning round needs the draft model");
  R.buckets = replan_buckets(n);
  SF_REQUIRE((int)R.buckets.size() <= kMaxBuckets, "too many Euler buckets");
  for (int bk : R.buckets) {
    Buffers* b = get_buffers(h, bk, 1, 1 | f32mode, &rc);
    if (!b) return rc;
    R.bb.push_back(b);
  }
  R.fbuckets = pol->mode_flash ? flash_buckets(n) : std::vector<int>{};
  SF_REQUIRE((int)R.fbuckets.size() <= kMaxBuckets, "too many flash buckets");
  for (int bk : R.fbuckets) {
    Buffers* b = bk == n ? nullptr : get_buffers(h, bk, cfg->k, f32mode, &rc);
    if (bk != n && !b) return rc;
    R.fbb.push_back(b);
  }
  if ((rc = dalloc(&R.eps_d, (size_t)n * hd)) || (rc = dalloc(&R.chunk, (size_t)n * hd)) ||
      (rc = dalloc(&R.chunk_raw, (size_t)n * hd)) || (rc = dalloc(&R.mean, (size_t)c.action_dim)) ||
      (rc = dalloc(&R.stdv, (size_t)c.action_dim)) || (rc = dalloc(&R.path, n)) ||
      (rc = dalloc(&R.planned, n)) || (rc = dalloc(&R.sie, n)) || (rc = dalloc(&R.bad, n)) ||
      (rc = dalloc(&R.fb_idx, n)) || (rc = dalloc(&R.fb_count, 1)) || (rc = dalloc(&R.use, n)) ||
      (rc = dalloc(&R.fl_idx, n)) || (rc = dalloc(&R.fl_count, 1)))
    return rc;
  if (pol->std_mean) {
    SF_CHECK_CUDA(cudaMemcpy(R.mean, pol->std_mean, sizeof(float) * c.action_dim, cudaMemcpyDeviceToDevice));
    SF_CHECK_CUDA(cudaMemcpy(R.stdv, pol->std_std, sizeof(float) * c.action_dim, cudaMemcpyDeviceToDevice));
  }
  if (!h.capture_stream)
    SF_CHECK_CUDA(cudaStreamCreateWithFlags(&h.capture_stream, cudaStreamNonBlocking));
  if (!h.body_stream) SF_CHECK_CUDA(cudaStreamCreateWithFlags(&h.body_stream, cudaStreamNonBlocking));
  cudaStream_t cs = h.capture_stream;
  Buffers& bf = *R.bf;
  const int64_t before = sf_launch_count(0);
  int64_t bodies = 0;  // kernels captured into SWITCH bodies (they run only when selected)
  cudaGraph_t g = nullptr;
  SF_CHECK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  auto fail = [&](int code) {
    cudaGraph_t junk = nullptr;
    cudaStreamEndCapture(cs, &junk);
    if (junk) cudaGraphDestroy(junk);
    sf::count_launch(-(int)(sf_launch_count(0) - before));
    return code;
  };
  auto begin_body = [&](cudaGraph_t body_graph, size_t i) {
    if (cudaStreamBeginCaptureToGraph(h.body_stream, body_graph, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      sf::set_error("body capture %zu failed", i);
      return SF_ECUDA;
    }
    return SF_OK;
  };
  // a bucket body's GEMMs / attention visit only the live rows / envs (the
  // compacted count on the device), not the bucket's padding; set for the
  // capture only (the Buffers are shared with the plain entry points)
  auto set_live = [&](Buffers& b, const int* cnt) {
    for (auto& op : b.ops) {
      op.p.rows_dev = cnt;
      op.p.rows_mul = b.env_rows;
    }
    b.ap.envs_dev = cnt;
  };
  auto end_body = [&](int brc, size_t i) {
    cudaGraph_t body = nullptr;
    const cudaError_t be = cudaStreamEndCapture(h.body_stream, &body);
    if (brc) return brc;
    if (be != cudaSuccess) {
      sf::set_error("body capture %zu: %s", i, cudaGetErrorString(be));
      return SF_ECUDA;
    }
    return SF_OK;
  };
  // 1. the speculative attempt of the envs that make one this round (a cached
  //    context, no forced periodic refresh: runtime.py:242-253), compacted into
  //    the smallest flash bucket (draft MLP -> verify -> gate -> decision); the
  //    results go back to the envs' rows of bf
  if (pol->mode_flash) {
    cudaGraphConditionalHandle fcond;
    if ((rc = make_switch_handle(cs, (int)R.fbuckets.size(), &fcond))) return fail(rc);
    FlashSelectParams fs{};
    fs.n = n;
    fs.fsr = fsr;
    fs.has_cache = has_cache;
    fs.mode_flash = pol->mode_flash;
    fs.pf = pol->periodic_refresh;
    fs.use = R.use;
    fs.fl_idx = R.fl_idx;
    fs.fl_count = R.fl_count;
    fs.n_buckets = (int)R.fbuckets.size();
    for (int i = 0; i < fs.n_buckets; ++i) fs.bucket[i] = R.fbuckets[i];
    fs.cond = fcond;
    flash_select_kernel<<<1, 1024, 0, cs>>>(fs);
    sf::count_launch(1);
    cudaGraphNodeParams fcp{};
    if ((rc = add_switch_node(cs, fcond, (int)R.fbuckets.size(), &fcp))) return fail(rc);
    for (size_t i = 0; i < R.fbuckets.size(); ++i) {
      if ((rc = begin_body(fcp.conditional.phGraph_out[i], i))) return fail(rc);
      cudaStream_t bs = h.body_stream;
      const int64_t k0 = sf_launch_count(0);
      int brc;
      if (!R.fbb[i]) {
        brc = enqueue_verify(h, bf, cfg, bs, pdl, true);  // every env attempts: in place
      } else {
        Buffers& b = *R.fbb[i];
        const int bk = R.fbuckets[i];
        FlashGatherParams gp{R.fl_idx, R.fl_count, bk, c.draft_in, hd, c.state_dim, bf.obs, bf.eps, bf.state,
                             bf.signs, b.obs, b.eps, b.state, b.signs, b.env_map};
        const int per = c.draft_in + hd + c.state_dim + 1;
        const int gblocks = (bk * per + 255) / 256 < 1184 ? (bk * per + 255) / 256 : 1184;
        flash_gather_kernel<<<gblocks, 256, 0, bs>>>(gp);
        sf::count_launch(1);
        set_live(b, R.fl_count);
        brc = enqueue_verify(h, b, cfg, bs, pdl, true);
        set_live(b, nullptr);
        FlashScatterParams sp{R.fl_idx, R.fl_count, cfg->k, hd, b.result, b.branch, b.draft,
                              bf.result, bf.branch, bf.draft};
        const int sper = SF_RESULT_WORDS + cfg->k + hd;
        const int sblocks = (bk * sper + 255) / 256 < 1184 ? (bk * sper + 255) / 256 : 1184;
        flash_scatter_kernel<<<sblocks, 256, 0, bs>>>(sp);
        sf::count_launch(1);
        R.flash_body_kernels = (int)(sf_launch_count(0) - k0);
      }
      bodies += sf_launch_count(0) - k0;
      if ((rc = end_body(brc, i))) return fail(rc);
    }
    flash_mark_kernel<<<(n * (SF_RESULT_WORDS + cfg->k) + 255) / 256, 256, 0, cs>>>(R.use, n, cfg->k, bf.result,
                                                                                 bf.branch);
    sf::count_launch(1);
  }
  // 2. bookkeeping + compaction + bucket select (sets the Euler SWITCH value)
  cudaGraphConditionalHandle cond;
  if ((rc = make_switch_handle(cs, (int)R.buckets.size(), &cond))) return fail(rc);
  ReplanSelectParams sp{};
  sp.n = n;
  sp.result = bf.result;
  sp.fsr = fsr;
  sp.has_cache = has_cache;
  sp.mode_flash = pol->mode_flash;
  sp.pf = pol->periodic_refresh;
  sp.r = cfg->replan_size;
  sp.path = R.path;
  sp.planned = R.planned;
  sp.fb_idx = R.fb_idx;
  sp.fb_count = R.fb_count;
  sp.n_buckets = (int)R.buckets.size();
  for (int i = 0; i < sp.n_buckets; ++i) sp.bucket[i] = R.buckets[i];
  sp.cond = cond;
  replan_select_kernel<<<1, 1024, 0, cs>>>(sp);
  chunk_init_kernel<<<(n * hd + 255) / 256 < 1184 ? (n * hd + 255) / 256 : 1184, 256, 0, cs>>>(
      bf.draft, R.chunk, R.bad, n, hd);
  sf::count_launch(2);
  // 3. SWITCH over the Euler buckets
  cudaGraphNodeParams cp{};
  if ((rc = add_switch_node(cs, cond, (int)R.buckets.size(), &cp))) return fail(rc);
  for (size_t i = 0; i < R.buckets.size(); ++i) {
    Buffers& b = *R.bb[i];
    const int bk = R.buckets[i];
    cudaStream_t bs = h.body_stream;
    if ((rc = begin_body(cp.conditional.phGraph_out[i], i))) return fail(rc);
    const int64_t k0 = sf_launch_count(0);
    const int per = hd + c.state_dim;
    const int gblocks = (bk * per + 255) / 256 < 1184 ? (bk * per + 255) / 256 : 1184;
    bucket_gather_kernel<<<gblocks, 256, 0, bs>>>(R.fb_idx, R.fb_count, bk, hd, c.state_dim, R.eps_d, bf.state,
                                                  b.draft, b.state, b.env_map);
    set_live(b, R.fb_count);
    int brc = enqueue_denoise(h, b, pol->num_steps, bs, pdl);
    set_live(b, nullptr);
    const int sblocks = (bk * hd + 255) / 256 < 1184 ? (bk * hd + 255) / 256 : 1184;
    bucket_scatter_kernel<<<sblocks, 256, 0, bs>>>(R.fb_idx, R.fb_count, hd, b.draft, b.status, R.chunk, R.bad);
    sf::count_launch(2);
    R.euler_body_kernels = (int)(sf_launch_count(0) - k0);
    bodies += sf_launch_count(0) - k0;
    if ((rc = end_body(brc, i))) return fail(rc);
  }
  // 4. non-finite flags, switch_in_executed, destandardize
  ReplanFinalParams fp{n, c.horizon, c.action_dim, R.path, R.planned, bf.result, bf.signs, R.chunk, R.bad,
                       R.sie, pol->std_mean ? R.chunk_raw : nullptr, R.mean, R.stdv};
  replan_finalize_kernel<<<(n * 32 + 255) / 256, 256, 0, cs>>>(fp);
  sf::count_launch(1);
  cudaError_t ce = cudaStreamEndCapture(cs, &g);
  R.fixed_kernels = (int)(sf_launch_count(0) - before - bodies);
  sf::count_launch(-(int)(sf_launch_count(0) - before));  // launched per replay, counted there
  if (ce != cudaSuccess) {
    sf::set_error("replan capture: %s", cudaGetErrorString(ce));
    if (g) cudaGraphDestroy(g);
    return SF_ECUDA;
  }
  ce = cudaGraphInstantiate(&R.exec, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) {
    sf::set_error("replan graph instantiate: %s", cudaGetErrorString(ce));
    R.exec = nullptr;
    return SF_ECUDA;
  }
  return SF_OK;
}

}  // namespace

extern "C" int sf_ae_replan_round(void* handle, int n_envs, const sf_verify_cfg_t* cfg,
                                  const sf_replan_policy_t* policy, const float* obs, const float* eps_verify,
                                  const float* eps_denoise, const float* state, const float* signs, int* fsr,
                                  int* has_cache, const sf_replan_out_t* out, int flags, void* stream) {
  auto* h = static_cast<Handle*>(handle);
  SF_REQUIRE(h && cfg && policy && obs && eps_verify && eps_denoise && state && signs && fsr && has_cache &&
                 out && out->chunk && out->path && out->planned,
             "null argument");
  SF_REQUIRE(h->k_prefix, "no prefix KV bound (sf_ae_set_prefix)");
  SF_REQUIRE(n_envs >= 1 && n_envs <= h->n_prefix_envs, "n_envs exceeds the prefix pool");
  SF_REQUIRE(policy->num_steps >= 1 && policy->num_steps <= 64, "num_steps must be in [1, 64]");
  SF_REQUIRE(policy->periodic_refresh >= 0, "periodic_refresh must be >= 0");
  SF_REQUIRE(!policy->std_mean == !policy->std_std, "standardizer needs both mean and std");
  int rc = check_verify_cfg(cfg, signs);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const sf_ae_config_t& c = h->cfg;
  if ((rc = ensure_temb(*h, cfg, s))) return rc;
  if ((rc = set_euler_steps(*h, policy->num_steps, s))) return rc;
  const bool pdl = (flags & SF_AE_PDL) != 0, fp32 = (flags & SF_AE_FP32) != 0;
  uint64_t key = 1469598103934665603ull;
  auto mix = [&](const void* q, size_t nb) {
    const unsigned char* b = static_cast<const unsigned char*>(q);
    for (size_t i = 0; i < nb; ++i) key = (key ^ b[i]) * 1099511628211ull;
  };
  const void* keyed[] = {fsr, has_cache, policy->std_mean, policy->std_std};
  const int knobs[] = {n_envs, cfg_key(cfg), policy->mode_flash, policy->periodic_refresh, policy->num_steps,
                       (int)pdl, (int)fp32};
  mix(keyed, sizeof(keyed));
  mix(knobs, sizeof(knobs));
  auto it = h->replans.find(key);
  if (it == h->replans.end()) {
    auto R = std::make_unique<Replan>();
    rc = build_replan(*h, *R, n_envs, cfg, policy, signs, fsr, has_cache, pdl, fp32);
    if (rc == SF_ECUDA && pdl) {  // programmatic edges inside conditional bodies unsupported: plain edges
      R = std::make_unique<Replan>();
      rc = build_replan(*h, *R, n_envs, cfg, policy, signs, fsr, has_cache, false, fp32);
    }
    if (rc) return rc;
    it = h->replans.emplace(key, std::move(R)).first;
  }
  Replan& R = *it->second;
  Buffers& bf = *R.bf;
  const size_t hd = (size_t)n_envs * c.horizon * c.action_dim;
  CopyList cin{};
  copy_list_add(cin, bf.obs, obs, (long long)n_envs * c.draft_in);
  copy_list_add(cin, bf.eps, eps_verify, (long long)hd);
  copy_list_add(cin, R.eps_d, eps_denoise, (long long)hd);
  copy_list_add(cin, bf.state, state, (long long)n_envs * c.state_dim);
  copy_list_add(cin, bf.signs, signs, n_envs);
  if ((rc = copy_list_launch(cin, s))) return rc;
  SF_CHECK_CUDA(cudaGraphLaunch(R.exec, s));
  sf::count_launch(R.fixed_kernels);
  h->replan_kernels[0] = R.fixed_kernels;
  h->replan_kernels[1] = R.flash_body_kernels ? R.flash_body_kernels - 2 : 0;
  h->replan_kernels[2] = R.euler_body_kernels;
  h->replan_kernels[3] = R.fbuckets.size() > 1 ? R.fbuckets[R.fbuckets.size() - 2] : 0;
  CopyList co{};
  copy_list_add(co, out->chunk, R.chunk, (long long)hd);
  if (out->chunk_raw && policy->std_mean) copy_list_add(co, out->chunk_raw, R.chunk_raw, (long long)hd);
  copy_list_add(co, out->path, R.path, n_envs);
  copy_list_add(co, out->planned, R.planned, n_envs);
  if (out->switch_in_executed) copy_list_add(co, out->switch_in_executed, R.sie, n_envs);
  if (out->nonfinite) copy_list_add(co, out->nonfinite, R.bad, n_envs);
  if (out->branch_prefixes) copy_list_add(co, out->branch_prefixes, bf.branch, (long long)n_envs * cfg->k);
  if (out->result) copy_list_add(co, out->result, bf.result, (long long)n_envs * SF_RESULT_WORDS);
  if (out->n_fallback) copy_list_add(co, out->n_fallback, R.fb_count, 1);
  return copy_list_launch(co, s);
}

extern "C" int sf_ae_replan_kernels(void* handle, int* out4) {
  auto* h = static_cast<Handle*>(handle);
  SF_REQUIRE(h && out4, "null argument");
  for (int i = 0; i < 4; ++i) out4[i] = h->replan_kernels[i];
  return SF_OK;
}

extern "C" int sf_ae_velocity(void* handle, int n_envs, int rows, const float* x, const double* taus,
                              const float* state, float* v_out, void* stream) {
  auto* h = static_cast<Handle*>(handle);
  SF_REQUIRE(h && x && taus && state && v_out, "null argument");
  SF_REQUIRE(h->k_prefix, "no prefix KV bound (sf_ae_set_prefix)");
  SF_REQUIRE(n_envs >= 1 && n_envs <= h->n_prefix_envs, "n_envs exceeds the prefix pool");
  SF_REQUIRE(rows >= 1 && rows <= SF_MAX_K, "rows must be in [1, %d]", SF_MAX_K);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = 0;
  Buffers* b = get_buffers(*h, n_envs, rows, 2, &rc);
  if (!b) return rc;
  sf_verify_cfg_t c{};
  c.k = rows;
  for (int r = 0; r < rows; ++r) {
    SF_REQUIRE(taus[r] >= 0.0 && taus[r] <= 1.0, "tau=%g outside [0, 1]", taus[r]);
    c.taus[r] = taus[r];
  }
  if ((rc = ensure_temb(*h, &c, s))) return rc;
  const sf_ae_config_t& cf = h->cfg;
  const size_t n = (size_t)n_envs * rows * cf.horizon * cf.action_dim;
  float* actions = nullptr;
  if ((rc = dalloc(&actions, n))) return rc;
  SF_CHECK_CUDA(cudaMemcpyAsync(actions, x, n * 4, cudaMemcpyDeviceToDevice, s));
  SF_CHECK_CUDA(cudaMemcpyAsync(b->state, state, (size_t)n_envs * cf.state_dim * 4,
                                cudaMemcpyDeviceToDevice, s));
  EmbedParams ep = embed_params(*h, *b, 1, h->temb);
  ep.draft = actions;
  if ((rc = launch_embed(b->M, h->cfg.width, s, ep, false))) return rc;
  if ((rc = run_stack(*h, *b, s, false))) return rc;
  GatherParams gp{b->vel, v_out, n_envs, rows, cf.horizon, cf.action_dim, T_of(*h), b->env_rows};
  gather_vel_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(gp);
  SF_CHECK_CUDA(cudaGetLastError());
  sf::count_launch();
  SF_CHECK_CUDA(cudaStreamSynchronize(s));
  cudaFree(actions);
  return SF_OK;
}

namespace sf {
namespace pi0 {

}  // namespace pi0
}  // namespace sf

// ===========================================================================
// Context refresh: VLM prefix prefill -> prefix KV pool (
// the pi0 analogue of encode_context, flowpolicy.py:156-161, runtime.py:166).
// A Gemma-style decoder stack (width W, 8 query heads x 256 sharing one KV
// head, GeGLU MLP, RMSNorm folded into the weights, RoPE) runs over the P
// prefix tokens of every env with bidirectional prefix attention, and its
// per-layer K / V are written straight into the pool layout the Action Expert
// attends to: K [L][E][P][256] (the QKV epilogue's row-major K output IS that
// layout) and V^T [L][E][256][P] (one transpose-copy per layer). Same kernels
// as the Action Expert: tcgen05 GEMMs (2-SM pairs at >= 1024 rows) with fused
// RMS/RoPE/residual/GeGLU epilogues, and the MQA attention kernel with
// prefix-only keys (segs = 0).
// ===========================================================================
namespace sf {
namespace pi0 {

struct VlmBuffers {
  int E = 0, M = 0, m_ld = 0;
  float* x = nullptr;
  bf16* xb = nullptr;
  float* ssq = nullptr;
  bf16* q = nullptr;
  bf16* vt = nullptr;  // [256][m_ld] V^T of the current layer
  bf16* attn = nullptr;
  bf16* h = nullptr;
  float* ws = nullptr;
  float* attn_ws = nullptr;
  int* counters = nullptr;
  int* env_ident = nullptr;
  std::vector<gemm::Op> ops;  // per layer: qkv, o, gu, down
  std::vector<CUtensorMap> maps;  // per layer: q, kp, vp, ks (dummy), vs (dummy)
  attn::Params ap{};
  int attn_tiles = 0, attn_splits = 1;
  void* k_pool = nullptr;
  void* vt_pool = nullptr;
};

struct VlmHandle {
  sf_vlm_config_t cfg{};
  sf_vlm_weights_t w{};
  float2* rope_t = nullptr;  // [128][P] position-fastest
  std::map<long long, std::unique_ptr<VlmBuffers>> buffers;
};

__global__ void prefill_embed_kernel(const float* __restrict__ x_in, float* x, bf16* xb, float* ssq,
                                     int M, int W, int ssq_ld) {
  // one warp per (row, 128-feature group)
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int groups = W / 128;
  if (warp >= M * groups) return;
  const int m = warp / groups, g = warp - m * groups;
  const float4 v = reinterpret_cast<const float4*>(x_in + (size_t)m * W + g * 128)[lane];
  reinterpret_cast<float4*>(x + (size_t)m * W + g * 128)[lane] = v;
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
  reinterpret_cast<uint2*>(xb + (size_t)m * W + g * 128)[lane] =
      make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  float sq = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0) ssq[(size_t)g * ssq_ld + m] = sq;
}

// V^T [256][m_ld] (env-major columns) -> pool slice [E][256][P]
__global__ void vt_to_pool_kernel(const bf16* __restrict__ vt, bf16* __restrict__ pool, int E, int P,
                                  int m_ld) {
  const size_t total = (size_t)E * 256 * P / 8;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t o = i * 8;  // pool element index (8 consecutive keys)
    const int p = (int)(o % P);
    const size_t ed = o / P;
    const int d = (int)(ed % 256), e = (int)(ed / 256);
    const bf16* src = vt + (size_t)d * m_ld + (size_t)e * P + p;
    bf16* dst = pool + o;
    if (p + 8 <= P && (P % 8) == 0) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
    } else {
      for (int z = 0; z < 8 && p + z < P; ++z) dst[z] = src[z];
    }
  }
}

int vlm_build(VlmHandle& h, VlmBuffers& b, int E, void* k_pool, void* vt_pool) {
  const sf_vlm_config_t& c = h.cfg;
  const int W = c.width, P = c.prefix_len, L = c.layers, nq = 8 * 256;
  b.E = E;
  b.M = E * P;
  b.m_ld = ((b.M + 63) / 64) * 64;
  b.k_pool = k_pool;
  b.vt_pool = vt_pool;
  int rc;
#define VALLOC(ptr, n) \
  if ((rc = dalloc(&(ptr), (n)))) return rc
  VALLOC(b.x, (size_t)b.M * W);
  VALLOC(b.xb, (size_t)b.m_ld * W);
  VALLOC(b.ssq, (size_t)(W / 128) * b.m_ld);
  VALLOC(b.q, (size_t)b.m_ld * nq);
  VALLOC(b.vt, (size_t)256 * b.m_ld);
  VALLOC(b.attn, (size_t)b.m_ld * nq);
  VALLOC(b.h, (size_t)b.m_ld * c.mlp);
  VALLOC(b.env_ident, (size_t)E);
  {
    std::vector<int> id(E);
    for (int i = 0; i < E; ++i) id[i] = i;
    SF_CHECK_CUDA(cudaMemcpy(b.env_ident, id.data(), sizeof(int) * E, cudaMemcpyHostToDevice));
  }
  auto epi_base = [&](int kind) {
    gemm::EpiArgs e{};
    e.kind = kind;
    e.M = b.M;
    e.ssq_in = b.ssq;
    e.ssq_groups = W / 128;
    e.ssq_ld = b.m_ld;
    e.inv_width = 1.f / (float)W;
    e.eps = c.eps;
    return e;
  };
  b.ops.resize(4 * L);
  const bool swap = b.M <= 256;
  const int bn = swap ? ((b.M + 15) / 16) * 16 : 256;
  auto plan_op = [&](gemm::Op* op, const void* wt, int n_out, const void* act, int k_in,
                     const gemm::EpiArgs& e) {
    if (swap) return gemm::plan(op, wt, n_out, k_in, act, b.M, k_in, k_in, bn, 0, 1, e);
    return gemm::plan(op, act, b.M, k_in, wt, n_out, k_in, k_in, bn, 1, 0, e);
  };
  for (int l = 0; l < L; ++l) {
    gemm::EpiArgs e = epi_base(gemm::EPI_QKV);
    e.N = nq + 512;
    e.q = b.q;
    e.k = static_cast<bf16*>(k_pool) + (size_t)l * E * P * 256;  // row m = e*P + p: pool layout
    e.vt = b.vt;
    e.vt_ld = b.m_ld;
    e.rope = h.rope_t;
    e.rope_ld = P;
    e.q_features = nq;
    e.env_rows = P;
    e.seg_len = P;
    e.pos0 = 0;
    if ((rc = plan_op(&b.ops[4 * l + 0], h.w.qkv[l], e.N, b.xb, W, e))) return rc;
    gemm::EpiArgs eo = epi_base(gemm::EPI_RESID);
    eo.ssq_in = nullptr;
    eo.N = W;
    eo.x = b.x;
    eo.xb = b.xb;
    eo.ssq_out = b.ssq;
    eo.ssq_out_ld = b.m_ld;
    if ((rc = plan_op(&b.ops[4 * l + 1], h.w.o[l], W, b.attn, nq, eo))) return rc;
    gemm::EpiArgs eg = epi_base(gemm::EPI_GEGLU);
    eg.N = 2 * c.mlp;
    eg.out_bf16 = b.h;
    eg.ld_bf16 = c.mlp;
    if ((rc = plan_op(&b.ops[4 * l + 2], h.w.gu[l], eg.N, b.xb, W, eg))) return rc;
    if ((rc = plan_op(&b.ops[4 * l + 3], h.w.down[l], W, b.h, c.mlp, eo))) return rc;
  }
  size_t need = 0;
  for (auto& op : b.ops) need = op.ws_bytes > need ? op.ws_bytes : need;
  if (need) {
    VALLOC(b.ws, need / sizeof(float));
    for (auto& op : b.ops) op.p.ws = b.ws;
  }
  // attention: prefix-only keys (segs = 0), bidirectional over the P tokens
  const int npb = (P + attn::BKEY - 1) / attn::BKEY;
  b.attn_tiles = b.M / 16;
  int asplit = 148 / b.attn_tiles;
  asplit = asplit < 1 ? 1 : (asplit > npb ? npb : asplit);
  asplit = asplit > attn::kMaxSplitsKV ? attn::kMaxSplitsKV : asplit;
  const int bps = (npb + asplit - 1) / asplit;
  asplit = (npb + bps - 1) / bps;
  b.attn_splits = asplit;
  if (asplit > 1) VALLOC(b.attn_ws, (size_t)b.attn_tiles * asplit * (attn::HD * attn::BQ + 2 * attn::BQ));
  VALLOC(b.counters, (size_t)b.attn_tiles + 8);
#undef VALLOC
  attn::Params& ap = b.ap;
  ap.M = b.M;
  ap.env_rows = P;
  ap.n_envs = E;
  ap.tiles_env = P / 16;
  ap.seg_len = P;
  ap.segs = 0;
  ap.prefix_len = P;
  ap.n_prefix_blocks = npb;
  ap.n_blocks = npb;
  ap.blocks_per_split = bps;
  ap.splits = asplit;
  ap.tiles = b.attn_tiles;
  ap.scale_log2 = 1.4426950408889634f / 16.f;
  ap.out = b.attn;
  ap.ws = b.attn_ws;
  ap.counters = b.counters;
  ap.env_map = b.env_ident;
  b.maps.resize(5 * L);
  for (int l = 0; l < L; ++l) {
    CUtensorMap* mp = &b.maps[5 * l];
    if ((rc = gemm::make_map(&mp[0], b.q, b.M * attn::kHeads, 256, 256, attn::BQ))) return rc;
    const bf16* kp = static_cast<const bf16*>(k_pool) + (size_t)l * E * P * 256;
    const bf16* vp = static_cast<const bf16*>(vt_pool) + (size_t)l * E * 256 * P;
    if ((rc = make_map_3d(&mp[1], kp, 256, P, E, 512, (uint64_t)P * 512, 64, attn::BKEY))) return rc;
    if ((rc = make_map_3d(&mp[2], vp, P, 256, E, (uint64_t)P * 2, (uint64_t)P * 512, attn::BKEY, 256)))
      return rc;
    // suffix maps are never used (no suffix blocks) but must be valid descriptors
    mp[3] = mp[0];
    mp[4] = mp[0];
  }
  return SF_OK;
}

int vlm_enqueue(VlmHandle& h, VlmBuffers& b, const float* x_in, cudaStream_t s) {
  const sf_vlm_config_t& c = h.cfg;
  const int L = c.layers, P = c.prefix_len;
  int rc;
  const int warps = b.M * (c.width / 128);
  prefill_embed_kernel<<<(warps * 32 + 255) / 256, 256, 0, s>>>(x_in, b.x, b.xb, b.ssq, b.M, c.width,
                                                                b.m_ld);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  static bool attr = false;
  if (!attr) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(attn::attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)attn::kSmemBytes));
    SF_CHECK_CUDA(cudaFuncSetAttribute(attn::attn_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  for (int l = 0; l < L; ++l) {
    if ((rc = gemm::launch(b.ops[4 * l + 0], s, false))) return rc;
    bf16* vpool = static_cast<bf16*>(b.vt_pool) + (size_t)l * b.E * 256 * P;
    vt_to_pool_kernel<<<148 * 4, 256, 0, s>>>(b.vt, vpool, b.E, P, b.m_ld);
    SF_CHECK_CUDA(cudaGetLastError());
    count_launch();
    const CUtensorMap* mp = &b.maps[5 * l];
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(b.attn_tiles, b.attn_splits);
    cfg.blockDim = dim3(attn::kThreads);
    cfg.dynamicSmemBytes = attn::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    int na = 0;
    if (b.attn_splits > 1) {
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = 1;
      a[0].val.clusterDim.y = b.attn_splits;
      a[0].val.clusterDim.z = 1;
      na = 1;
    }
    cfg.attrs = a;
    cfg.numAttrs = na;
    SF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, attn::attn_kernel, mp[0], mp[1], mp[2], mp[3], mp[4], b.ap));
    count_launch();
    if ((rc = gemm::launch(b.ops[4 * l + 1], s, false))) return rc;
    if ((rc = gemm::launch(b.ops[4 * l + 2], s, false))) return rc;
    if ((rc = gemm::launch(b.ops[4 * l + 3], s, false))) return rc;
  }
  return SF_OK;
}

}  // namespace pi0
}  // namespace sf

using sf::pi0::VlmBuffers;
using sf::pi0::VlmHandle;

extern "C" int sf_vlm_create(const sf_vlm_config_t* cfg, const sf_vlm_weights_t* w, void** handle) {
  SF_REQUIRE(cfg && w && handle, "null argument");
  SF_REQUIRE(cfg->q_heads == 8 && cfg->head_dim == 256, "the attention kernel is built for 8 x 256 MQA");
  SF_REQUIRE(cfg->width % 256 == 0 && cfg->width <= 4096, "width must be a multiple of 256 (<= 4096)");
  SF_REQUIRE(cfg->layers >= 1 && cfg->layers <= SF_AE_MAX_LAYERS, "bad layer count");
  SF_REQUIRE(cfg->mlp % 128 == 0, "mlp must be a multiple of 128");
  SF_REQUIRE(cfg->prefix_len >= 16 && cfg->prefix_len % 16 == 0, "prefix_len must be a multiple of 16");
  auto* h = new VlmHandle();
  h->cfg = *cfg;
  h->w = *w;
  int rc;
  if ((rc = sf::pi0::dalloc(&h->rope_t, (size_t)128 * cfg->prefix_len))) {
    delete h;
    return rc;
  }
  sf::pi0::transpose_u64_kernel<<<64, 256>>>(static_cast<const unsigned long long*>(w->rope),
                                             reinterpret_cast<unsigned long long*>(h->rope_t),
                                             cfg->prefix_len, 128);
  SF_CHECK_CUDA(cudaGetLastError());
  SF_CHECK_CUDA(cudaDeviceSynchronize());
  *handle = h;
  return SF_OK;
}

extern "C" int sf_vlm_destroy(void* handle) {
  auto* h = static_cast<VlmHandle*>(handle);
  if (!h) return SF_OK;
  for (auto& kv : h->buffers) {
    VlmBuffers& b = *kv.second;
    void* ptrs[] = {b.x, b.xb, b.ssq, b.q, b.vt, b.attn, b.h, b.ws, b.attn_ws, b.counters, b.env_ident};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
  cudaFree(h->rope_t);
  delete h;
  return SF_OK;
}

extern "C" int sf_vlm_prefill(void* handle, int n_envs, const float* x, void* k_pool, void* vt_pool,
                              void* stream) {
  auto* h = static_cast<VlmHandle*>(handle);
  SF_REQUIRE(h && x && k_pool && vt_pool && n_envs >= 1, "bad prefill arguments");
  cudaStream_t s = (cudaStream_t)stream;
  // plans embed the pool pointers: key on (envs, pools)
  const long long key = (long long)n_envs ^ ((long long)(uintptr_t)k_pool << 8) ^
                        ((long long)(uintptr_t)vt_pool << 20);
  auto it = h->buffers.find(key);
  VlmBuffers* b;
  if (it == h->buffers.end()) {
    auto nb = std::make_unique<VlmBuffers>();
    int rc = sf::pi0::vlm_build(*h, *nb, n_envs, k_pool, vt_pool);
    if (rc) return rc;
    b = nb.get();
    h->buffers[key] = std::move(nb);
  } else {
    b = it->second.get();
  }
  return sf::pi0::vlm_enqueue(*h, *b, x, s);
}
