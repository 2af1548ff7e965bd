// Tiny-model speculative-replanning kernels (cfg1/cfg2/cfg5, batch 1).
//
// B200 design: the whole round is ONE launch of one thread-block cluster
// (kCluster CTAs x 256 threads). Every MLP layer is split across all CTAs of
// the cluster by output neuron; each warp owns one output row of W at a time
// (coalesced row stream from L2, K rows of activations from SMEM) and pushes
// the finished activation into every CTA's SMEM through DSMEM, followed by one
// cluster barrier per layer. The round is latency-bound (1.4 MB of weights,
// 1.7 MFLOP) so the design minimises launches and global round trips: draft
// MLP -> K-branch interpolation/packing -> field MLP -> reconstruction ->
// distances -> warp-ballot prefix scan -> gripper gate -> decision all happen
// inside the same launch; the Euler full path keeps its N steps inside one
// launch too.
//
// Reference semantics: nets.py:90-107 (MLP), flowpolicy.py:196-209 (packing,
// endpoint field), verifier.py:65-150 (Alg. 1), actions.py:168-211 (distance,
// gate), runtime.py:286-320 (decision), flowpolicy.py:273-292 (Euler).

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sf {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kCluster = 8;
constexpr int kMaxRows = 8;  // K rows per field evaluation (cfg5 sweeps K <= 8)

template <typename T>
struct DevMlp {
  int n_layers;
  int sizes[SF_MAX_LAYERS + 1];
  const T* w[SF_MAX_LAYERS];
  const T* b[SF_MAX_LAYERS];
};

template <typename T>
DevMlp<T> to_dev(const sf_mlp_t* m) {
  DevMlp<T> d{};
  if (!m) return d;
  d.n_layers = m->n_layers;
  for (int i = 0; i <= m->n_layers; ++i) d.sizes[i] = m->sizes[i];
  for (int i = 0; i < m->n_layers; ++i) {
    d.w[i] = static_cast<const T*>(m->w[i]);
    d.b[i] = static_cast<const T*>(m->b[i]);
  }
  return d;
}

// One MLP layer for `rows` activation rows, distributed over the cluster.
// in:  this CTA's SMEM [rows][n_in];  out: [rows][n_out] in EVERY CTA's SMEM.
template <typename T>
__device__ void cluster_layer(cg::cluster_group& cluster, const T* __restrict__ W,
                              const T* __restrict__ bias, int n_in, int n_out, int rows,
                              const T* in, T* out, bool tanh_act) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int csize = (int)cluster.num_blocks();
  const int gwarp = (int)cluster.block_rank() * kWarps + warp;
  const int total = csize * kWarps;
  for (int j = gwarp; j < n_out; j += total) {
    T acc[kMaxRows];
#pragma unroll
    for (int r = 0; r < kMaxRows; ++r) acc[r] = T(0);
    const T* wr = W + (size_t)j * n_in;
    for (int i = lane; i < n_in; i += 32) {
      const T w = __ldg(wr + i);
#pragma unroll
      for (int r = 0; r < kMaxRows; ++r)
        if (r < rows) acc[r] = fma(w, in[r * n_in + i], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < kMaxRows; ++r) {
      if (r < rows) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], off);
      }
    }
    T mine = T(0);
#pragma unroll
    for (int r = 0; r < kMaxRows; ++r)
      if (r == lane) mine = acc[r];
    // z = a @ W.T + b, tanh on hidden layers (nets.py:103-104)
    T z = add_rn(mine, __ldg(bias + j));
    if (tanh_act) z = tanh_t(z);
    // row r's value lives in lane r; lane c pushes it into CTA c's SMEM (DSMEM)
    for (int r = 0; r < rows; ++r) {
      const T v = __shfl_sync(0xffffffffu, z, r);
      for (int c = lane; c < csize; c += 32) {
        T* dst = cluster.map_shared_rank(out, c);
        dst[r * n_out + j] = v;
      }
    }
  }
  cluster.sync();
}

// Whole MLP; ping-pongs between bufA (input, row stride sizes[0]) and bufB.
// Returns the buffer that holds the output.
template <typename T>
__device__ T* cluster_mlp(cg::cluster_group& cluster, const DevMlp<T>& m, int rows, T* bufA,
                          T* bufB) {
  T* in = bufA;
  T* out = bufB;
  for (int l = 0; l < m.n_layers; ++l) {
    cluster_layer<T>(cluster, m.w[l], m.b[l], m.sizes[l], m.sizes[l + 1], rows, in, out,
                     l + 1 < m.n_layers);
    T* t = in;
    in = out;
    out = t;
  }
  return in;
}

template <typename T>
struct FlashParams {
  DevMlp<T> draft;
  int has_draft;
  const T* draft_in;
  DevMlp<T> field;
  const T* emb;
  int emb_dim;
  const T* state;
  int state_dim;
  const T* eps;
  int H, D, C;
  int K;
  T taus[SF_MAX_K];
  T delta;
  int metric, window;
  T sign;
  int phase_fallback, prefix_cap, replan_size;
  T* out_draft;
  T* out_recon;
  T* out_dist;
  int* out_branch;
  int* out_result;
  int buf_elems;  // elements per ping-pong buffer
};

// Shared verification epilogue (one CTA): interpolate, reconstruct
// x + (1 - tau) v with v = (out - x) / (1 - tau) for endpoint nets
// (flowpolicy.py:209, verifier.py:88) or v given, distances, per-branch prefix
// via warp ballots, min over K, gripper gate over draft + branches, decision.
// `net_out(k, i)` returns the field net output (endpoint) or velocity.
template <typename T, bool kEndpoint, typename NetOut>
__device__ void verify_epilogue_cta(const T* draft, const T* eps, NetOut&& net_out, int H, int D,
                                    int C, int K, const T* taus, T delta, int metric, int window,
                                    T sign, int phase_fallback, int prefix_cap, int replan_size,
                                    T* out_recon, T* out_dist, int* out_branch, int* out_result,
                                    T* s_recon /* smem [K*H*D] */, T* s_dist /* smem [K*H] */) {
  __shared__ int s_nonfinite;
  __shared__ int s_switch;
  __shared__ int s_branch[SF_MAX_K];
  if (threadIdx.x == 0) {
    s_nonfinite = 0x7fffffff;
    s_switch = 0;
  }
  __syncthreads();
  const int HD = H * D;
  for (int idx = threadIdx.x; idx < K * HD; idx += blockDim.x) {
    const int k = idx / HD, i = idx - k * HD;
    const T tau = taus[k];
    const T omt = sub_rn(T(1), tau);
    // interpolate: tau * draft + (1 - tau) * eps (verifier.py:73)
    const T x = add_rn(mul_rn(tau, draft[i]), mul_rn(omt, eps[i]));
    T v;
    if (kEndpoint) {
      v = div_rn(sub_rn(net_out(k, i), x), omt);
    } else {
      v = net_out(k, i);
    }
    const T recon = add_rn(x, mul_rn(omt, v));
    if (!finite_t(v) || !finite_t(recon)) atomicMin(&s_nonfinite, k);
    s_recon[idx] = recon;
    if (out_recon) out_recon[idx] = recon;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < K * H; idx += blockDim.x) {
    const int k = idx / H, h = idx - k * H;
    const T* a = draft + h * D;
    const T* b = s_recon + (size_t)k * HD + h * D;
    const T d = step_distance<T>(C, metric, [&](int c) { return a[c]; },
                                 [&](int c) { return b[c]; });
    s_dist[idx] = d;
    if (out_dist) out_dist[idx] = d;
  }
  // gripper gate: any(g[:window] * sign <= 0) over draft and every branch
  const int win = window < 0 ? H : (window < H ? window : H);
  for (int idx = threadIdx.x; idx < (K + 1) * win; idx += blockDim.x) {
    const int c = idx / win, h = idx - c * win;
    const T g = c == 0 ? draft[h * D + D - 1] : s_recon[(size_t)(c - 1) * HD + h * D + D - 1];
    if (mul_rn(g, sign) <= T(0)) s_switch = 1;  // benign race: all writers store 1
  }
  __syncthreads();
  // prefix per branch: first h with !(d <= delta); warp k scans branch k
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < K; k += blockDim.x >> 5) {
    int prefix = H;
    for (int base = 0; base < H; base += 32) {
      const int h = base + lane;
      const bool fail = h < H && !(s_dist[k * H + h] <= delta);
      const unsigned m = __ballot_sync(0xffffffffu, fail);
      if (m) {
        prefix = base + __ffs(m) - 1;
        break;
      }
    }
    if (lane == 0) s_branch[k] = prefix;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int L = H;
    for (int k = 0; k < K; ++k) {
      L = min(L, s_branch[k]);
      out_branch[k] = s_branch[k];
    }
    const int sw = s_switch;
    const bool phase_fb = phase_fallback && sw;
    const bool rejected = L == 0;
    int path, planned;
    if (phase_fb || rejected) {
      path = phase_fb ? SF_PATH_FLASH_PHASE : SF_PATH_FLASH_REJECTED;
      planned = replan_size;
    } else {
      path = SF_PATH_FLASH_ACCEPTED;
      const int cap = prefix_cap ? replan_size : H;
      planned = min(L, cap);
    }
    out_result[SF_RES_PREFIX] = L;
    out_result[SF_RES_SWITCH] = sw;
    out_result[SF_RES_PATH] = path;
    out_result[SF_RES_PLANNED] = planned;
    out_result[SF_RES_NONFINITE] = s_nonfinite == 0x7fffffff ? -1 : s_nonfinite;
  }
}

template <typename T>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads, 1)
    tiny_flash_round_kernel(const FlashParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  T* bufA = reinterpret_cast<T*>(smem_raw);
  T* bufB = bufA + p.buf_elems;
  T* s_draft = bufB + p.buf_elems;
  const int HD = p.H * p.D;

  // ---- 1. draft (draft.py:57-61): one MLP forward on the feature vector
  const T* draft_vals;
  if (p.has_draft) {
    const int f = p.draft.sizes[0];
    for (int i = threadIdx.x; i < f; i += blockDim.x) bufA[i] = p.draft_in[i];
    __syncthreads();
    cluster.sync();  // remote writes of layer 0 must not race a slow CTA's setup
    const T* o = cluster_mlp<T>(cluster, p.draft, 1, bufA, bufB);
    for (int i = threadIdx.x; i < HD; i += blockDim.x) s_draft[i] = o[i];
    __syncthreads();
    draft_vals = s_draft;
  } else {
    draft_vals = p.draft_in;
  }
  if (cluster.block_rank() == 0 && p.out_draft)
    for (int i = threadIdx.x; i < HD; i += blockDim.x) p.out_draft[i] = draft_vals[i];

  // ---- 2. pack K rows [x_k, tau_k, emb, state] (flowpolicy.py:196-201)
  const int n_in = p.field.sizes[0];
  for (int idx = threadIdx.x; idx < p.K * n_in; idx += blockDim.x) {
    const int k = idx / n_in, i = idx - k * n_in;
    const T tau = p.taus[k];
    T v;
    if (i < HD)
      v = add_rn(mul_rn(tau, draft_vals[i]), mul_rn(sub_rn(T(1), tau), p.eps[i]));
    else if (i == HD)
      v = tau;
    else if (i < HD + 1 + p.emb_dim)
      v = p.emb[i - HD - 1];
    else
      v = p.state[i - HD - 1 - p.emb_dim];
    bufA[idx] = v;
  }
  __syncthreads();
  cluster.sync();

  // ---- 3. field MLP over the K branches as one K-row batch
  const T* out = cluster_mlp<T>(cluster, p.field, p.K, bufA, bufB);

  // ---- 4. epilogue on rank 0 (distances, prefix, gate, decision)
  if (cluster.block_rank() == 0) {
    T* s_recon = const_cast<T*>(out == bufA ? bufB : bufA);  // free buffer
    T* s_dist = s_recon + p.K * HD;
    verify_epilogue_cta<T, true>(
        draft_vals, p.eps, [&](int k, int i) { return out[k * HD + i]; }, p.H, p.D, p.C, p.K,
        p.taus, p.delta, p.metric, p.window, p.sign, p.phase_fallback, p.prefix_cap,
        p.replan_size, p.out_recon, p.out_dist, p.out_branch, p.out_result, s_recon, s_dist);
  }
}

template <typename T>
struct FullParams {
  DevMlp<T> enc;
  int has_enc;
  const T* enc_in;
  int emb_dim;
  DevMlp<T> field;
  const T* state;
  int state_dim;
  const T* start;
  int H, D, N;
  T* out_chunk;
  T* out_emb;
  int* status;
  int buf_elems;
};

template <typename T>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads, 1)
    tiny_full_round_kernel(const FullParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  T* bufA = reinterpret_cast<T*>(smem_raw);
  T* bufB = bufA + p.buf_elems;
  T* s_emb = bufB + p.buf_elems;
  T* s_vals = s_emb + p.emb_dim;
  __shared__ int s_bad;
  __shared__ int s_bad_v;
  const int HD = p.H * p.D;

  // ---- encode_context: emb = [features, MLP(features)] (flowpolicy.py:143-147)
  if (p.has_enc) {
    const int f = p.enc.sizes[0];
    for (int i = threadIdx.x; i < f; i += blockDim.x) {
      bufA[i] = p.enc_in[i];
      s_emb[i] = p.enc_in[i];
    }
    __syncthreads();
    cluster.sync();
    const T* o = cluster_mlp<T>(cluster, p.enc, 1, bufA, bufB);
    const int fo = p.enc.sizes[p.enc.n_layers];
    for (int i = threadIdx.x; i < fo; i += blockDim.x) s_emb[f + i] = o[i];
  } else {
    for (int i = threadIdx.x; i < p.emb_dim; i += blockDim.x) s_emb[i] = p.enc_in[i];
  }
  for (int i = threadIdx.x; i < HD; i += blockDim.x) s_vals[i] = p.start[i];
  if (threadIdx.x == 0) {
    s_bad = -1;
    s_bad_v = 0;
  }
  __syncthreads();
  if (cluster.block_rank() == 0 && p.out_emb)
    for (int i = threadIdx.x; i < p.emb_dim; i += blockDim.x) p.out_emb[i] = s_emb[i];

  // ---- Euler: tau_i = i/N, A <- A + v(A, tau)/N (flowpolicy.py:286-291)
  const int n_in = p.field.sizes[0];
  for (int step = 0; step < p.N; ++step) {
    const T tau = (T)((double)step / (double)p.N);
    for (int i = threadIdx.x; i < n_in; i += blockDim.x) {
      T v;
      if (i < HD) v = s_vals[i];
      else if (i == HD) v = tau;
      else if (i < HD + 1 + p.emb_dim) v = s_emb[i - HD - 1];
      else v = p.state[i - HD - 1 - p.emb_dim];
      bufA[i] = v;
    }
    __syncthreads();
    cluster.sync();
    const T* out = cluster_mlp<T>(cluster, p.field, 1, bufA, bufB);
    const T omt = sub_rn(T(1), tau);
    const T n = (T)p.N;
    for (int i = threadIdx.x; i < HD; i += blockDim.x) {
      const T a = s_vals[i];
      const T vel = div_rn(sub_rn(out[i], a), omt);  // flowpolicy.py:209
      const T nxt = add_rn(a, div_rn(vel, n));        // flowpolicy.py:289
      if (!finite_t(vel)) atomicOr(&s_bad_v, 1);
      if (!finite_t(nxt) && s_bad < 0) atomicCAS(&s_bad, -1, step);
      s_vals[i] = nxt;
    }
    __syncthreads();
    if (s_bad >= 0) break;  // the reference raises at the first bad step
  }
  if (cluster.block_rank() == 0) {
    for (int i = threadIdx.x; i < HD; i += blockDim.x) p.out_chunk[i] = s_vals[i];
    if (threadIdx.x == 0 && p.status) {
      p.status[0] = s_bad;
      p.status[1] = s_bad_v;
    }
  }
}


template <typename T>
struct EvalParams {
  DevMlp<T> field;
  const T* x;  // [R, HD]
  T taus[kMaxRows];
  int R;
  const T* emb;
  int emb_dim;
  const T* state;
  int state_dim;
  int HD;
  T* out_v;
  int* status;  // [R]: 1 if v non-finite
  int buf_elems;
};

// Field protocol evaluation (flowpolicy.py:203-209): R rows packed
// [x_r, tau_r, emb, state] through the endpoint net, v = (out - x)/(1 - tau).
template <typename T>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads, 1)
    tiny_field_eval_kernel(const EvalParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  T* bufA = reinterpret_cast<T*>(smem_raw);
  T* bufB = bufA + p.buf_elems;
  const int n_in = p.field.sizes[0];
  for (int idx = threadIdx.x; idx < p.R * n_in; idx += blockDim.x) {
    const int r = idx / n_in, i = idx - r * n_in;
    T v;
    if (i < p.HD) v = p.x[r * p.HD + i];
    else if (i == p.HD) v = p.taus[r];
    else if (i < p.HD + 1 + p.emb_dim) v = p.emb[i - p.HD - 1];
    else v = p.state[i - p.HD - 1 - p.emb_dim];
    bufA[idx] = v;
  }
  __syncthreads();
  cluster.sync();
  const T* out = cluster_mlp<T>(cluster, p.field, p.R, bufA, bufB);
  if (cluster.block_rank() != 0) return;
  __shared__ int s_bad[kMaxRows];
  if (threadIdx.x < kMaxRows) s_bad[threadIdx.x] = 0;
  __syncthreads();
  for (int idx = threadIdx.x; idx < p.R * p.HD; idx += blockDim.x) {
    const int r = idx / p.HD;
    const T x = p.x[idx];
    const T v = div_rn(sub_rn(out[idx], x), sub_rn(T(1), p.taus[r]));
    if (!finite_t(v)) s_bad[r] = 1;
    p.out_v[idx] = v;
  }
  __syncthreads();
  if (threadIdx.x < p.R && p.status) p.status[threadIdx.x] = s_bad[threadIdx.x];
}

template <typename T>
struct FwdParams {
  DevMlp<T> net;
  const T* x;  // [R, n_in]
  int R;
  T* out;      // [R, n_out]
  int buf_elems;
};

// Plain MLP forward for R <= 8 rows (nets.forward, nets.py:90-107).
template <typename T>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads, 1)
    tiny_mlp_forward_kernel(const FwdParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  T* bufA = reinterpret_cast<T*>(smem_raw);
  T* bufB = bufA + p.buf_elems;
  const int n_in = p.net.sizes[0], n_out = p.net.sizes[p.net.n_layers];
  for (int i = threadIdx.x; i < p.R * n_in; i += blockDim.x) bufA[i] = p.x[i];
  __syncthreads();
  cluster.sync();
  const T* o = cluster_mlp<T>(cluster, p.net, p.R, bufA, bufB);
  if (cluster.block_rank() == 0)
    for (int i = threadIdx.x; i < p.R * n_out; i += blockDim.x) p.out[i] = o[i];
}

// ------------------------------------------------ field-agnostic kernels

struct Taus {
  double v[SF_MAX_K];
};

template <typename T>
__global__ void interpolate_kernel(const T* draft, const T* eps, const Taus taus, int K, int n,
                                   T* out) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < K * n; idx += gridDim.x * blockDim.x) {
    const int k = idx / n, i = idx - k * n;
    const T tau = (T)taus.v[k];
    out[idx] = add_rn(mul_rn(tau, draft[i]), mul_rn(sub_rn(T(1), tau), eps[i]));
  }
}

template <typename T>
struct EpiParams {
  const T* draft;
  const T* eps;
  const T* vel;
  int H, D, C, K;
  T taus[SF_MAX_K];
  T delta;
  int metric, window;
  T sign;
  int phase_fallback, prefix_cap, replan_size;
  T* out_recon;
  T* out_dist;
  int* out_branch;
  int* out_result;
};

template <typename T>
__global__ void __launch_bounds__(kThreads) verify_epilogue_kernel(const EpiParams<T> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_recon = reinterpret_cast<T*>(smem_raw);
  T* s_dist = s_recon + p.K * p.H * p.D;
  const int HD = p.H * p.D;
  verify_epilogue_cta<T, false>(
      p.draft, p.eps, [&](int k, int i) { return p.vel[k * HD + i]; }, p.H, p.D, p.C, p.K, p.taus,
      p.delta, p.metric, p.window, p.sign, p.phase_fallback, p.prefix_cap, p.replan_size,
      p.out_recon, p.out_dist, p.out_branch, p.out_result, s_recon, s_dist);
}

// One warp per row: first index with !(d <= delta) via ballots.
template <typename T>
__global__ void prefix_kernel(const T* d, int rows, int h, T delta, int* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const T* row = d + (size_t)warp * h;
  int prefix = h;
  for (int base = 0; base < h; base += 32) {
    const int i = base + lane;
    const unsigned m = __ballot_sync(0xffffffffu, i < h && !(row[i] <= delta));
    if (m) {
      prefix = base + __ffs(m) - 1;
      break;
    }
  }
  if (lane == 0) out[warp] = prefix;
}

template <typename T>
__global__ void distance_kernel(const T* a, const T* b, int rows, int D, int C, int metric, T* out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const T* ar = a + (size_t)r * D;
    const T* br = b + (size_t)r * D;
    out[r] = step_distance<T>(C, metric, [&](int c) { return ar[c]; }, [&](int c) { return br[c]; });
  }
}

template <typename T>
__global__ void gripper_kernel(const T* v, int n_chunks, int H, int D, T sign, int window, int* out) {
  const int win = window < 0 ? H : (window < H ? window : H);
  int hit = 0;
  for (int idx = threadIdx.x; idx < n_chunks * win; idx += blockDim.x) {
    const int c = idx / win, h = idx - c * win;
    if (mul_rn(v[((size_t)c * H + h) * D + D - 1], sign) <= T(0)) hit = 1;
  }
  hit = __syncthreads_or(hit);
  if (threadIdx.x == 0) out[0] = hit;
}

template <typename T>
__global__ void euler_update_kernel(T* vals, const T* vel, int count, int n, int step, int* status) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const T nxt = add_rn(vals[i], div_rn(vel[i], (T)n));
    vals[i] = nxt;
    if (!finite_t(nxt)) atomicCAS(status, -1, step);
  }
}

template <typename T>
int check_cfg_copy(const sf_verify_cfg_t* cfg, T* taus, int H) {
  SF_REQUIRE(cfg, "null verifier config");
  SF_REQUIRE(cfg->k >= 1 && cfg->k <= SF_MAX_K, "need 1..%d verification timesteps, got %d",
             SF_MAX_K, cfg->k);
  for (int i = 0; i < cfg->k; ++i) {
    SF_REQUIRE(cfg->taus[i] > 0.0 && cfg->taus[i] < 1.0,
               "verification timesteps must lie strictly inside (0, 1)");
    if (i) SF_REQUIRE(cfg->taus[i] > cfg->taus[i - 1], "verification timesteps must be strictly increasing");
    taus[i] = (T)cfg->taus[i];
  }
  SF_REQUIRE(cfg->delta >= 0.0, "delta must be non-negative");
  SF_REQUIRE(cfg->metric == SF_METRIC_L2 || cfg->metric == SF_METRIC_LINF, "unknown metric");
  SF_REQUIRE(cfg->current_sign == 1.0 || cfg->current_sign == -1.0,
             "current_sign must be -1.0 or +1.0");
  SF_REQUIRE(cfg->replan_size >= 1, "replan_size must be >= 1");
  (void)H;
  return SF_OK;
}

int mlp_max_width(const sf_mlp_t* m) {
  int w = 0;
  for (int i = 0; m && i <= m->n_layers; ++i) w = w > m->sizes[i] ? w : m->sizes[i];
  return w;
}

int check_mlp(const sf_mlp_t* m, const char* name) {
  SF_REQUIRE(m->n_layers >= 1 && m->n_layers <= SF_MAX_LAYERS, "%s: bad layer count %d", name,
             m->n_layers);
  for (int i = 0; i < m->n_layers; ++i) {
    SF_REQUIRE(m->w[i] && m->b[i], "%s: null weights in layer %d", name, i);
    SF_REQUIRE(m->sizes[i] > 0 && m->sizes[i + 1] > 0, "%s: bad sizes", name);
  }
  return SF_OK;
}

template <typename T>
int flash_round_impl(const sf_mlp_t* draft_net, const void* draft_in, const sf_mlp_t* field_net,
                     const void* emb, int emb_dim, const void* state, int state_dim,
                     const void* eps, int H, int D, int C, const sf_verify_cfg_t* cfg,
                     const sf_verify_out_t* out, cudaStream_t stream) {
  FlashParams<T> p{};
  int rc = check_cfg_copy<T>(cfg, p.taus, H);
  if (rc) return rc;
  SF_REQUIRE(field_net && draft_in && eps && out && out->branch_prefixes && out->result,
             "null argument");
  if ((rc = check_mlp(field_net, "field"))) return rc;
  SF_REQUIRE(cfg->k <= kMaxRows, "tiny path supports K <= %d", kMaxRows);
  SF_REQUIRE(H >= 1 && D >= 2 && C >= 1 && C <= D - 1, "bad chunk shape H=%d D=%d C=%d", H, D, C);
  SF_REQUIRE(field_net->sizes[0] == H * D + 1 + emb_dim + state_dim,
             "velocity net dimensions do not match (H, D, emb, state)");
  SF_REQUIRE(field_net->sizes[field_net->n_layers] == H * D, "field output must be H*D");
  if (draft_net) {
    if ((rc = check_mlp(draft_net, "draft"))) return rc;
    SF_REQUIRE(draft_net->sizes[draft_net->n_layers] == H * D,
               "draft net output does not match horizon x dim");
  }
  p.draft = to_dev<T>(draft_net);
  p.has_draft = draft_net != nullptr;
  p.draft_in = static_cast<const T*>(draft_in);
  p.field = to_dev<T>(field_net);
  p.emb = static_cast<const T*>(emb);
  p.emb_dim = emb_dim;
  p.state = static_cast<const T*>(state);
  p.state_dim = state_dim;
  p.eps = static_cast<const T*>(eps);
  p.H = H;
  p.D = D;
  p.C = C;
  p.K = cfg->k;
  p.delta = (T)cfg->delta;
  p.metric = cfg->metric;
  p.window = cfg->window;
  p.sign = (T)cfg->current_sign;
  p.phase_fallback = cfg->phase_fallback;
  p.prefix_cap = cfg->prefix_cap;
  p.replan_size = cfg->replan_size;
  p.out_draft = static_cast<T*>(out->draft);
  p.out_recon = static_cast<T*>(out->reconstructed);
  p.out_dist = static_cast<T*>(out->distances);
  p.out_branch = out->branch_prefixes;
  p.out_result = out->result;
  int width = mlp_max_width(field_net);
  if (draft_net) width = width > mlp_max_width(draft_net) ? width : mlp_max_width(draft_net);
  const int rows = cfg->k;
  // ping-pong buffers must also host the epilogue's recon [K*H*D] + dist [K*H]
  int buf = width * rows;
  const int epi = rows * H * D + rows * H;
  buf = buf > epi ? buf : epi;
  p.buf_elems = (buf + 3) & ~3;
  const size_t smem = sizeof(T) * ((size_t)2 * p.buf_elems + H * D + 4);
  SF_REQUIRE(smem <= 220 * 1024, "tiny round needs %zu B of shared memory (max 220 KB)", smem);
  auto kern = tiny_flash_round_kernel<T>;
  SF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<kCluster, kThreads, smem, stream>>>(p);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}

template <typename T>
int full_round_impl(const sf_mlp_t* enc, const void* enc_in, int emb_dim, const sf_mlp_t* field_net,
                    const void* state, int state_dim, const void* start, int H, int D, int N,
                    void* chunk_out, void* emb_out, int* status, cudaStream_t stream) {
  int rc;
  SF_REQUIRE(enc_in && start && chunk_out, "null argument");
  SF_REQUIRE(N >= 0, "num_steps must be >= 0");
  SF_REQUIRE(field_net || N == 0, "null field");
  if (N > 0 && (rc = check_mlp(field_net, "field"))) return rc;
  if (enc) {
    if ((rc = check_mlp(enc, "encoder"))) return rc;
    SF_REQUIRE(enc->sizes[0] + enc->sizes[enc->n_layers] == emb_dim,
               "encoder embed_dim (in + out) must equal emb_dim");
  }
  if (N > 0) {
    SF_REQUIRE(field_net->sizes[0] == H * D + 1 + emb_dim + state_dim,
               "velocity net dimensions do not match (H, D, emb, state)");
    SF_REQUIRE(field_net->sizes[field_net->n_layers] == H * D, "field output must be H*D");
  }
  FullParams<T> p{};
  p.enc = to_dev<T>(enc);
  p.has_enc = enc != nullptr;
  p.enc_in = static_cast<const T*>(enc_in);
  p.emb_dim = emb_dim;
  p.field = to_dev<T>(field_net);
  p.state = static_cast<const T*>(state);
  p.state_dim = state_dim;
  p.start = static_cast<const T*>(start);
  p.H = H;
  p.D = D;
  p.N = N;
  p.out_chunk = static_cast<T*>(chunk_out);
  p.out_emb = static_cast<T*>(emb_out);
  p.status = status;
  int width = mlp_max_width(field_net);
  if (enc) width = width > mlp_max_width(enc) ? width : mlp_max_width(enc);
  p.buf_elems = (width + 3) & ~3;
  const size_t smem = sizeof(T) * ((size_t)2 * p.buf_elems + emb_dim + H * D + 4);
  SF_REQUIRE(smem <= 220 * 1024, "tiny full round needs %zu B of shared memory", smem);
  auto kern = tiny_full_round_kernel<T>;
  SF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<kCluster, kThreads, smem, stream>>>(p);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}

template <typename T>
int field_eval_impl(const sf_mlp_t* field_net, const void* x, const double* taus, int R,
                    const void* emb, int emb_dim, const void* state, int state_dim, int H, int D,
                    void* out_v, int* status, cudaStream_t stream) {
  int rc;
  SF_REQUIRE(field_net && x && taus && out_v, "null argument");
  SF_REQUIRE(R >= 1 && R <= kMaxRows, "field evaluation supports 1..%d rows", kMaxRows);
  if ((rc = check_mlp(field_net, "field"))) return rc;
  SF_REQUIRE(field_net->sizes[0] == H * D + 1 + emb_dim + state_dim,
             "velocity net dimensions do not match (H, D, emb, state)");
  SF_REQUIRE(field_net->sizes[field_net->n_layers] == H * D, "field output must be H*D");
  EvalParams<T> p{};
  p.field = to_dev<T>(field_net);
  p.x = static_cast<const T*>(x);
  for (int r = 0; r < R; ++r) {
    SF_REQUIRE(taus[r] >= 0.0 && taus[r] <= 1.0, "tau=%g outside [0, 1]", taus[r]);
    p.taus[r] = (T)taus[r];
  }
  p.R = R;
  p.emb = static_cast<const T*>(emb);
  p.emb_dim = emb_dim;
  p.state = static_cast<const T*>(state);
  p.state_dim = state_dim;
  p.HD = H * D;
  p.out_v = static_cast<T*>(out_v);
  p.status = status;
  p.buf_elems = (mlp_max_width(field_net) * R + 3) & ~3;
  const size_t smem = sizeof(T) * (size_t)2 * p.buf_elems;
  SF_REQUIRE(smem <= 220 * 1024, "field evaluation needs %zu B of shared memory", smem);
  auto kern = tiny_field_eval_kernel<T>;
  SF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<kCluster, kThreads, smem, stream>>>(p);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}

template <typename T>
int mlp_forward_impl(const sf_mlp_t* net, const void* x, int R, void* out, cudaStream_t stream) {
  int rc;
  SF_REQUIRE(net && x && out, "null argument");
  SF_REQUIRE(R >= 1 && R <= kMaxRows, "mlp forward supports 1..%d rows", kMaxRows);
  if ((rc = check_mlp(net, "mlp"))) return rc;
  FwdParams<T> p{};
  p.net = to_dev<T>(net);
  p.x = static_cast<const T*>(x);
  p.R = R;
  p.out = static_cast<T*>(out);
  p.buf_elems = (mlp_max_width(net) * R + 3) & ~3;
  const size_t smem = sizeof(T) * (size_t)2 * p.buf_elems;
  SF_REQUIRE(smem <= 220 * 1024, "mlp forward needs %zu B of shared memory", smem);
  auto kern = tiny_mlp_forward_kernel<T>;
  SF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<kCluster, kThreads, smem, stream>>>(p);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}

template <typename T>
int epilogue_impl(const void* draft, const void* eps, const void* vel, int H, int D, int C,
                  const sf_verify_cfg_t* cfg, const sf_verify_out_t* out, cudaStream_t stream) {
  EpiParams<T> p{};
  int rc = check_cfg_copy<T>(cfg, p.taus, H);
  if (rc) return rc;
  SF_REQUIRE(draft && eps && vel && out && out->branch_prefixes && out->result, "null argument");
  SF_REQUIRE(H >= 1 && D >= 2 && C >= 1 && C <= D - 1, "bad chunk shape");
  p.draft = static_cast<const T*>(draft);
  p.eps = static_cast<const T*>(eps);
  p.vel = static_cast<const T*>(vel);
  p.H = H;
  p.D = D;
  p.C = C;
  p.K = cfg->k;
  p.delta = (T)cfg->delta;
  p.metric = cfg->metric;
  p.window = cfg->window;
  p.sign = (T)cfg->current_sign;
  p.phase_fallback = cfg->phase_fallback;
  p.prefix_cap = cfg->prefix_cap;
  p.replan_size = cfg->replan_size;
  p.out_recon = static_cast<T*>(out->reconstructed);
  p.out_dist = static_cast<T*>(out->distances);
  p.out_branch = out->branch_prefixes;
  p.out_result = out->result;
  const size_t smem = sizeof(T) * ((size_t)cfg->k * H * D + (size_t)cfg->k * H);
  SF_REQUIRE(smem <= 220 * 1024, "verify epilogue needs %zu B of shared memory", smem);
  auto kern = verify_epilogue_kernel<T>;
  SF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<1, kThreads, smem, stream>>>(p);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}

}  // namespace
}  // namespace sf

using sf::count_launch;

#define SF_DISPATCH(prec, FN, ...)                                   \
  ((prec) == SF_F32 ? FN<float>(__VA_ARGS__)                         \
   : (prec) == SF_F64 ? FN<double>(__VA_ARGS__)                      \
                      : (::sf::set_error("unknown precision %d", prec), SF_EINVAL))

extern "C" int sf_tiny_flash_round(int precision, const sf_mlp_t* draft_net, const void* draft_in,
                                   const sf_mlp_t* field_net, const void* emb, int emb_dim,
                                   const void* state, int state_dim, const void* eps, int horizon,
                                   int dim, int continuous_dims, const sf_verify_cfg_t* cfg,
                                   const sf_verify_out_t* out, void* stream) {
  return SF_DISPATCH(precision, sf::flash_round_impl, draft_net, draft_in, field_net, emb, emb_dim,
                     state, state_dim, eps, horizon, dim, continuous_dims, cfg, out,
                     (cudaStream_t)stream);
}

extern "C" int sf_tiny_full_round(int precision, const sf_mlp_t* encoder, const void* enc_in,
                                  int emb_dim, const sf_mlp_t* field_net, const void* state,
                                  int state_dim, const void* start, int horizon, int dim,
                                  int num_steps, void* chunk_out, void* emb_out, int* status,
                                  void* stream) {
  return SF_DISPATCH(precision, sf::full_round_impl, encoder, enc_in, emb_dim, field_net, state,
                     state_dim, start, horizon, dim, num_steps, chunk_out, emb_out, status,
                     (cudaStream_t)stream);
}

extern "C" int sf_tiny_mlp_forward(int precision, const sf_mlp_t* net, const void* x, int rows,
                                   void* out, void* stream) {
  return SF_DISPATCH(precision, sf::mlp_forward_impl, net, x, rows, out, (cudaStream_t)stream);
}

extern "C" int sf_tiny_field_eval(int precision, const sf_mlp_t* field_net, const void* x,
                                  const double* taus, int rows, const void* emb, int emb_dim,
                                  const void* state, int state_dim, int horizon, int dim,
                                  void* velocity_out, int* status, void* stream) {
  return SF_DISPATCH(precision, sf::field_eval_impl, field_net, x, taus, rows, emb, emb_dim, state,
                     state_dim, horizon, dim, velocity_out, status, (cudaStream_t)stream);
}

extern "C" int sf_verify_epilogue(int precision, const void* draft, const void* eps,
                                  const void* velocity, int horizon, int dim, int continuous_dims,
                                  const sf_verify_cfg_t* cfg, const sf_verify_out_t* out,
                                  void* stream) {
  return SF_DISPATCH(precision, sf::epilogue_impl, draft, eps, velocity, horizon, dim,
                     continuous_dims, cfg, out, (cudaStream_t)stream);
}

namespace sf {
namespace {
template <typename T>
int interpolate_impl(const void* draft, const void* eps, const double* taus, int k, int n, void* out,
                     cudaStream_t stream) {
  SF_REQUIRE(draft && eps && taus && out && k >= 1 && k <= SF_MAX_K && n >= 1,
             "bad interpolate arguments");
  Taus t{};
  for (int i = 0; i < k; ++i) {
    SF_REQUIRE(taus[i] >= 0.0 && taus[i] <= 1.0, "tau=%g outside [0, 1]", taus[i]);
    t.v[i] = taus[i];
  }
  interpolate_kernel<T><<<(k * n + 255) / 256, 256, 0, stream>>>(
      static_cast<const T*>(draft), static_cast<const T*>(eps), t, k, n, static_cast<T*>(out));
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}
template <typename T>
int prefix_impl(const void* d, int rows, int h, double delta, int* out, cudaStream_t stream) {
  SF_REQUIRE(d && out && rows >= 0 && h >= 0, "bad prefix_length arguments");
  if (rows == 0) return SF_OK;
  const int threads = 256, warps = threads / 32;
  prefix_kernel<T><<<(rows + warps - 1) / warps, threads, 0, stream>>>(static_cast<const T*>(d),
                                                                        rows, h, (T)delta, out);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}
template <typename T>
int distance_impl(const void* a, const void* b, int rows, int D, int C, int metric, void* out,
                  cudaStream_t stream) {
  SF_REQUIRE(a && b && out && rows >= 0 && C >= 0 && C <= D, "bad distance arguments");
  SF_REQUIRE(metric == SF_METRIC_L2 || metric == SF_METRIC_LINF, "unknown metric");
  if (rows == 0) return SF_OK;
  distance_kernel<T><<<(rows + 255) / 256, 256, 0, stream>>>(
      static_cast<const T*>(a), static_cast<const T*>(b), rows, D, C, metric, static_cast<T*>(out));
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}
template <typename T>
int gripper_impl(const void* v, int n_chunks, int H, int D, double sign, int window, int* out,
                 cudaStream_t stream) {
  SF_REQUIRE(sign == 1.0 || sign == -1.0, "current_sign must be -1.0 or +1.0");
  SF_REQUIRE(v && out && n_chunks >= 1 && H >= 1 && D >= 1, "bad gripper arguments");
  gripper_kernel<T><<<1, 256, 0, stream>>>(static_cast<const T*>(v), n_chunks, H, D, (T)sign,
                                           window, out);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}
template <typename T>
int euler_impl(void* vals, const void* vel, int count, int n, int step, int* status,
               cudaStream_t stream) {
  SF_REQUIRE(vals && vel && status && count >= 1 && n >= 1, "bad euler arguments");
  euler_update_kernel<T><<<(count + 255) / 256, 256, 0, stream>>>(
      static_cast<T*>(vals), static_cast<const T*>(vel), count, n, step, status);
  SF_CHECK_CUDA(cudaGetLastError());
  count_launch();
  return SF_OK;
}
}  // namespace
}  // namespace sf

extern "C" int sf_interpolate(int precision, const void* draft, const void* eps, const double* taus,
                              int k, int n, void* out, void* stream) {
  return SF_DISPATCH(precision, sf::interpolate_impl, draft, eps, taus, k, n, out,
                     (cudaStream_t)stream);
}
extern "C" int sf_prefix_length(int precision, const void* distances, int rows, int h, double delta,
                                int* out, void* stream) {
  return SF_DISPATCH(precision, sf::prefix_impl, distances, rows, h, delta, out,
                     (cudaStream_t)stream);
}
extern "C" int sf_continuous_distances(int precision, const void* a, const void* b, int rows,
                                       int dim, int continuous_dims, int metric, void* out,
                                       void* stream) {
  return SF_DISPATCH(precision, sf::distance_impl, a, b, rows, dim, continuous_dims, metric, out,
                     (cudaStream_t)stream);
}
extern "C" int sf_gripper_switch(int precision, const void* values, int n_chunks, int horizon,
                                 int dim, double current_sign, int window, int* out, void* stream) {
  return SF_DISPATCH(precision, sf::gripper_impl, values, n_chunks, horizon, dim, current_sign,
                     window, out, (cudaStream_t)stream);
}
extern "C" int sf_euler_update(int precision, void* values, const void* velocity, int count, int n,
                               int step, int* status, void* stream) {
  return SF_DISPATCH(precision, sf::euler_impl, values, velocity, count, n, step, status,
                     (cudaStream_t)stream);
}
