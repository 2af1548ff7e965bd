// Tiny-model speculative-replanning kernels (cfg1/cfg2/cfg5, batch 1).
//
// B200 design. The round is latency-bound (1.4 MB of weights, 1.7 MFLOP), so
// it runs as ONE launch of one thread-block cluster (16 CTAs x 256 threads
// when the GPU schedules 16-CTA clusters, else 8):
//  * At launch every CTA issues TMA bulk copies (cp.async.bulk, one mbarrier
//    per layer) of ITS row slice of EVERY layer of every net into SMEM, so the
//    whole model streams from L2/HBM in parallel across the cluster while the
//    first layer computes; the Euler full path then reuses the SMEM-resident
//    weights for all N steps. Layers that do not fit stay in global memory and
//    are streamed with unrolled loads.
//  * Each layer is split across the cluster by output neuron; a warp owns one
//    output row at a time (K activation rows from SMEM), reduces with
//    shuffles and pushes the activation into every CTA's SMEM with
//    st.async (DSMEM stores that complete_tx on the receiver's mbarrier).
//    A layer ends when the CTA's own output buffer has received all bytes --
//    no cluster barrier per layer (cluster.sync() compiles to MEMBAR.ALL.GPU
//    + the cluster barrier, ~0.8 us per layer measured). Three activation
//    buffers rotate so that a layer's pushes only target a buffer every CTA
//    has finished reading (see cluster_mlp).
//  * The speculative round fuses draft MLP -> K-branch interpolation/packing
//    -> field MLP -> reconstruction -> distances -> warp-ballot prefix scan ->
//    gripper gate -> decision; the full round fuses encoder -> N Euler steps.
//
// Reference: nets.py:90-107 (MLP), flowpolicy.py:196-209 (packing, endpoint
// field), verifier.py:65-150 (Alg. 1), actions.py:168-211, runtime.py:286-320,
// flowpolicy.py:273-292 (Euler).

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "sm100.cuh"
#include "verify_epi.cuh"

namespace cg = cooperative_groups;

namespace sf {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRows = 8;  // branch rows per field evaluation (cfg5 sweeps K <= 8)
constexpr size_t kSmemBudget = 224 * 1024;

template <typename T>
struct DevMlp {
  int n_layers;
  int sizes[SF_MAX_LAYERS + 1];
  int ld[SF_MAX_LAYERS];
  const T* w[SF_MAX_LAYERS];
  const T* b[SF_MAX_LAYERS];
  int woff[SF_MAX_LAYERS];  // element offset of this CTA's slice in the SMEM arena; -1 = global
};

template <typename T>
DevMlp<T> to_dev(const sf_mlp_t* m) {
  DevMlp<T> d{};
  if (!m) return d;
  d.n_layers = m->n_layers;
  for (int i = 0; i <= m->n_layers; ++i) d.sizes[i] = m->sizes[i];
  for (int i = 0; i < m->n_layers; ++i) {
    d.ld[i] = m->ld[i] > 0 ? m->ld[i] : m->sizes[i];
    d.w[i] = static_cast<const T*>(m->w[i]);
    d.b[i] = static_cast<const T*>(m->b[i]);
    d.woff[i] = -1;
  }
  return d;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          sm100::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(sm100::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void slice_rows(int n_out, int rank, int csize, int& r0, int& r1) {
  const int rpc = (n_out + csize - 1) / csize;
  r0 = min(n_out, rank * rpc);
  r1 = min(n_out, r0 + rpc);
}

// Issue the TMA bulk copies of this CTA's weight slices (all resident layers).
template <typename T>
__device__ void stage_weights(const DevMlp<T>& m, T* arena, uint64_t* bars, int rank, int csize) {
  if (threadIdx.x != 0) return;
  for (int l = 0; l < m.n_layers; ++l) {
    if (m.woff[l] < 0) continue;
    int r0, r1;
    slice_rows(m.sizes[l + 1], rank, csize, r0, r1);
    if (r1 <= r0) continue;
    const uint32_t bytes = (uint32_t)((size_t)(r1 - r0) * m.ld[l] * sizeof(T));
    sm100::mbar_arrive_expect_tx(&bars[l], bytes);
    bulk_g2s(arena + m.woff[l], m.w[l] + (size_t)r0 * m.ld[l], bytes, &bars[l]);
  }
}

template <typename T>
__device__ void init_bars(const DevMlp<T>& m, uint64_t* bars) {
  if (threadIdx.x != 0) return;
  for (int l = 0; l < m.n_layers; ++l)
    if (m.woff[l] >= 0) sm100::mbar_init(&bars[l], 1);
}


// Optional trace (sf_tiny_trace): %globaltimer stamps of rank 0, thread 0.
__device__ int g_tiny_trace_on = 0;
__device__ unsigned long long g_tiny_trace[32];
__device__ __forceinline__ void tstamp(int k) {
  if (g_tiny_trace_on && threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tiny_trace[k] = t;
  }
}

// SMEM map shared by all cluster kernels:
//   [bars: 2 nets x SF_MAX_LAYERS u64][bufA][bufB][extra][weight arena]
template <typename T>
struct Frame {
  uint64_t* bars0;
  uint64_t* bars1;
  uint64_t* full;  // [3] activation buffer i received all of a layer's pushes
  T* buf0;         // activation buffer i at buf0 + i * stride (no indexed array: it
  int stride;      // would live on the stack)
  T* extra;
  T* arena;
  __device__ T* buf(int i) const { return buf0 + i * stride; }
};

constexpr int kFrameBars = 2 * SF_MAX_LAYERS + 4;

template <typename T>
__device__ Frame<T> frame(unsigned char* smem, int buf_elems, int extra_elems) {
  Frame<T> f;
  f.bars0 = reinterpret_cast<uint64_t*>(smem);
  f.bars1 = f.bars0 + SF_MAX_LAYERS;
  f.full = f.bars1 + SF_MAX_LAYERS;
  f.buf0 = reinterpret_cast<T*>(smem + kFrameBars * sizeof(uint64_t));
  f.stride = buf_elems;
  f.extra = f.buf0 + 3 * buf_elems;
  f.arena = f.extra + extra_elems;
  return f;
}

template <typename T>
size_t frame_bytes(int buf_elems, int extra_elems) {
  return kFrameBars * sizeof(uint64_t) + sizeof(T) * ((size_t)3 * buf_elems + extra_elems);
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// DSMEM store that signals `bytes` on the receiving CTA's mbarrier
__device__ __forceinline__ void st_async(uint32_t addr, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr),
               "r"(__float_as_uint(v)), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(bar)
               : "memory");
}

// One layer for `rows` activation rows. in: this CTA's SMEM [rows][n_in];
// out: f.buf(oi) [rows][n_out] of EVERY CTA (st.async push). Returns after
// this CTA's own f.buf(oi) holds the whole layer output. `ph` carries the
// phase bits of the three full barriers (identical in every thread).
template <typename T, int ROWS>
__device__ void cluster_layer(cg::cluster_group& cluster, const Frame<T>& f, const DevMlp<T>& m, int l,
                              uint64_t* bars, const T* in, int oi, uint32_t& ph) {
  constexpr int rows = ROWS;  // compile-time: no predicated lanes / divergent shuffles
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster.block_rank(), csize = (int)cluster.num_blocks();
  const int n_in = m.sizes[l], n_out = m.sizes[l + 1], ld = m.ld[l];
  const bool resident = m.woff[l] >= 0;
  const bool act = l + 1 < m.n_layers;
  const T* arena = f.arena;
  // arm this layer's fill of my output buffer (its previous fill was consumed
  // before the previous layer; early remote bytes only make tx-count negative)
  if (threadIdx.x == 0) sm100::mbar_arrive_expect_tx(&f.full[oi], (uint32_t)(rows * n_out * sizeof(T)));
  int r0, r1;
  slice_rows(n_out, rank, csize, r0, r1);
  // lane c < csize pushes to CTA c
  uint32_t rout = 0, rbar = 0;
  if (lane < csize) {
    rout = mapa_u32(sm100::smem_u32(f.buf(oi)), (uint32_t)lane);
    rbar = mapa_u32(sm100::smem_u32(&f.full[oi]), (uint32_t)lane);
  }
  if (resident && r1 > r0) sm100::mbar_wait(&bars[l], 0);
  for (int j = r0 + warp; j < r1; j += kWarps) {
    const T bias = __ldg(m.b[l] + j);  // in flight during the dot products
    T acc[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) acc[r] = T(0);
    if (resident) {
      const T* wr = arena + m.woff[l] + (size_t)(j - r0) * ld;
      for (int i = lane; i < n_in; i += 32) {
        const T w = wr[i];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) acc[r] = fma(w, in[r * n_in + i], acc[r]);
      }
    } else {
      const T* wr = m.w[l] + (size_t)j * ld;
      int i = lane;
      for (; i + 96 < n_in; i += 128) {  // 4 independent loads in flight per lane
        const T w0 = __ldg(wr + i), w1 = __ldg(wr + i + 32), w2 = __ldg(wr + i + 64),
                w3 = __ldg(wr + i + 96);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          const T* a = in + r * n_in + i;
          acc[r] = fma(w0, a[0], acc[r]);
          acc[r] = fma(w1, a[32], acc[r]);
          acc[r] = fma(w2, a[64], acc[r]);
          acc[r] = fma(w3, a[96], acc[r]);
        }
      }
      for (; i < n_in; i += 32) {
        const T w = __ldg(wr + i);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) acc[r] = fma(w, in[r * n_in + i], acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], off);
    }
    T mine = T(0);
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
      if (r == lane) mine = acc[r];
    T z = add_rn(mine, bias);  // z = a @ W.T + b (nets.py:103)
    if (act) z = tanh_t(z);    // tanh on hidden layers (nets.py:104)
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const T v = __shfl_sync(0xffffffffu, z, r);
      if (lane < csize) st_async(rout + (uint32_t)((r * n_out + j) * sizeof(T)), v, rbar);
    }
  }
  sm100::mbar_wait(&f.full[oi], (ph >> oi) & 1u);
  ph ^= 1u << oi;
}

// Whole MLP on input `in` (ready in this CTA: received, or filled locally and
// __syncthreads'd). Layer 0 pushes into buffer o0, layer 1 into a1, then they
// alternate. The rotation is race-free when a1 is the buffer holding `in` and
// o0 is a buffer no CTA still reads: layer s >= 1 pushes into the input of
// layer s - 1, and a CTA pushes layer s only after it received every CTA's
// layer s - 1 output, i.e. after every CTA finished reading that input.
// Returns the index of the buffer holding the output.
template <typename T>
__device__ int cluster_mlp(cg::cluster_group& cluster, const Frame<T>& f, const DevMlp<T>& m, uint64_t* bars,
                           int rows, const T* in, int o0, int a1, uint32_t& ph) {
  int oi = o0;
  for (int l = 0; l < m.n_layers; ++l) {
    switch (rows) {
#define SF_ROWS_CASE(R) \
  case R: cluster_layer<T, R>(cluster, f, m, l, bars, in, oi, ph); break;
      SF_ROWS_CASE(1) SF_ROWS_CASE(2) SF_ROWS_CASE(3) SF_ROWS_CASE(4)
      SF_ROWS_CASE(5) SF_ROWS_CASE(6) SF_ROWS_CASE(7) SF_ROWS_CASE(8)
#undef SF_ROWS_CASE
      default: __trap();
    }
    tstamp(8 + l + (rows > 1 ? 8 : 0));
    in = f.buf(oi);
    oi = (oi == o0) ? a1 : o0;
  }
  return (oi == o0) ? a1 : o0;
}

// Prologue: barrier init, weight staging for up to two nets, cluster-wide
// start barrier (DSMEM must not be touched before every CTA runs).
template <typename T>
__device__ void prologue(cg::cluster_group& cluster, const Frame<T>& f, const DevMlp<T>& n0,
                         const DevMlp<T>* n1) {
  init_bars(n0, f.bars0);
  if (n1) init_bars(*n1, f.bars1);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) sm100::mbar_init(&f.full[i], 1);
    sm100::fence_barrier_init();
  }
  __syncthreads();
  const int rank = (int)cluster.block_rank(), csize = (int)cluster.num_blocks();
  stage_weights(n0, f.arena, f.bars0, rank, csize);
  if (n1) stage_weights(*n1, f.arena, f.bars1, rank, csize);
  // biases are read per output row in cluster_layer (global loads here would
  // serialise ~1 us of latency per layer into the prologue)
}

// ------------------------------------------------------------ flash round

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
  int H, D, C, K;
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
  int buf_elems, extra_elems;
};

template <typename T>
__global__ void __launch_bounds__(kThreads, 1) tiny_flash_round_kernel(const FlashParams<T> p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const Frame<T> f = frame<T>(smem_raw, p.buf_elems, p.extra_elems);
  T* s_draft = f.extra;
  const int HD = p.H * p.D;
  tstamp(0);
  prologue<T>(cluster, f, p.field, p.has_draft ? &p.draft : nullptr);
  tstamp(1);

  uint32_t ph = 0;
  // 1. draft (draft.py:57-61)
  const T* draft_vals;
  if (p.has_draft) {
    for (int i = threadIdx.x; i < p.draft.sizes[0]; i += blockDim.x) f.buf(0)[i] = p.draft_in[i];
    __syncthreads();
    cluster.sync();  // every CTA's barriers are initialised before the first push
    const int oi = cluster_mlp<T>(cluster, f, p.draft, f.bars1, 1, f.buf(0), 1, 0, ph);
    for (int i = threadIdx.x; i < HD; i += blockDim.x) s_draft[i] = f.buf(oi)[i];
    __syncthreads();
    draft_vals = s_draft;
  } else {
    cluster.sync();
    draft_vals = p.draft_in;
  }
  if (cluster.block_rank() == 0 && p.out_draft)
    for (int i = threadIdx.x; i < HD; i += blockDim.x) p.out_draft[i] = draft_vals[i];

  // 2. K packed rows [x_k, tau_k, emb, state] (flowpolicy.py:196-201)
  const int n_in = p.field.sizes[0];
  for (int idx = threadIdx.x; idx < p.K * n_in; idx += blockDim.x) {
    const int k = idx / n_in, i = idx - k * n_in;
    const T tau = p.taus[k];
    T v;
    if (i < HD) v = add_rn(mul_rn(tau, draft_vals[i]), mul_rn(sub_rn(T(1), tau), p.eps[i]));
    else if (i == HD) v = tau;
    else if (i < HD + 1 + p.emb_dim) v = p.emb[i - HD - 1];
    else v = p.state[i - HD - 1 - p.emb_dim];
    f.buf(0)[idx] = v;  // no push targets buffer 0 until every CTA finished field layer 0
  }
  __syncthreads();
  tstamp(2);

  // 3. field MLP over the K branches as one K-row batch; layer 0 pushes into
  // buffer 2 (never used before), so a CTA still copying the draft output out
  // of buffer 1 is not overwritten
  const int fo = cluster_mlp<T>(cluster, f, p.field, f.bars0, p.K, f.buf(0), 2, 0, ph);
  const T* out = f.buf(fo);

  // 4. epilogue on rank 0
  if (cluster.block_rank() == 0) {
    T* s_recon = f.buf(fo == 1 ? 0 : 1);
    T* s_dist = s_recon + p.K * HD;
    verify_epilogue_cta<T, true>(
        draft_vals, p.eps, [&](int k, int i) { return out[k * HD + i]; }, p.H, p.D, p.C, p.K,
        p.taus, p.delta, p.metric, p.window, p.sign, p.phase_fallback, p.prefix_cap,
        p.replan_size, p.out_recon, p.out_dist, p.out_branch, p.out_result, s_recon, s_dist);
  }
  tstamp(3);
  cluster.sync();  // no CTA exits while its pushes to peers may be in flight
}

// ------------------------------------------------------------- full round

template <typename T>
struct FullParams {
  DevMlp<T> enc;
  int has_enc;
  const T* enc_in;
  int emb_dim;
  DevMlp<T> field;
  int has_field;
  const T* state;
  int state_dim;
  const T* start;
  int H, D, N;
  T* out_chunk;
  T* out_emb;
  int* status;
  int buf_elems, extra_elems;
};

template <typename T>
__global__ void __launch_bounds__(kThreads, 1) tiny_full_round_kernel(const FullParams<T> p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const Frame<T> f = frame<T>(smem_raw, p.buf_elems, p.extra_elems);
  T* s_emb = f.extra;
  T* s_vals = s_emb + p.emb_dim;
  T* s_state = s_vals + p.H * p.D;
  __shared__ int s_bad, s_bad_v;
  const int HD = p.H * p.D;
  prologue<T>(cluster, f, p.field, p.has_enc ? &p.enc : nullptr);

  // encode_context: emb = [features, MLP(features)] (flowpolicy.py:143-147)
  uint32_t ph = 0;
  int last = 2;  // buffer holding the previous MLP's output (read by lagging CTAs)
  if (p.has_enc) {
    const int fi = p.enc.sizes[0];
    for (int i = threadIdx.x; i < fi; i += blockDim.x) {
      f.buf(0)[i] = p.enc_in[i];
      s_emb[i] = p.enc_in[i];
    }
    __syncthreads();
    cluster.sync();  // every CTA's barriers are initialised before the first push
    last = cluster_mlp<T>(cluster, f, p.enc, f.bars1, 1, f.buf(0), 1, 0, ph);
    for (int i = threadIdx.x; i < p.enc.sizes[p.enc.n_layers]; i += blockDim.x) s_emb[fi + i] = f.buf(last)[i];
  } else {
    for (int i = threadIdx.x; i < p.emb_dim; i += blockDim.x) s_emb[i] = p.enc_in[i];
    cluster.sync();
  }
  for (int i = threadIdx.x; i < HD; i += blockDim.x) s_vals[i] = p.start[i];
  for (int i = threadIdx.x; i < p.state_dim; i += blockDim.x) s_state[i] = p.state[i];
  if (threadIdx.x == 0) {
    s_bad = -1;
    s_bad_v = 0;
  }
  __syncthreads();
  if (cluster.block_rank() == 0 && p.out_emb)
    for (int i = threadIdx.x; i < p.emb_dim; i += blockDim.x) p.out_emb[i] = s_emb[i];

  // Euler: tau_i = i/N, A <- A + v(A, tau)/N (flowpolicy.py:286-291); every
  // CTA holds identical values, so the early exit is cluster-uniform.
  const int n_in = p.has_field ? p.field.sizes[0] : 0;
  for (int step = 0; step < p.N; ++step) {
    const T tau = (T)((double)step / (double)p.N);
    const int pin = (last + 1) % 3;  // no push targets it before every CTA finished layer 0
    for (int i = threadIdx.x; i < n_in; i += blockDim.x) {
      T v;
      if (i < HD) v = s_vals[i];
      else if (i == HD) v = tau;
      else if (i < HD + 1 + p.emb_dim) v = s_emb[i - HD - 1];
      else v = s_state[i - HD - 1 - p.emb_dim];
      f.buf(pin)[i] = v;
    }
    __syncthreads();
    // layer 0 pushes into the third buffer: neither the one a lagging CTA may
    // still read (the previous output) nor the packed input
    last = cluster_mlp<T>(cluster, f, p.field, f.bars0, 1, f.buf(pin), (last + 2) % 3, pin, ph);
    const T* out = f.buf(last);
    const T omt = sub_rn(T(1), tau);
    const T n = (T)p.N;
    for (int i = threadIdx.x; i < HD; i += blockDim.x) {
      const T a = s_vals[i];
      const T vel = div_rn(sub_rn(out[i], a), omt);  // flowpolicy.py:209
      const T nxt = add_rn(a, div_rn(vel, n));        // flowpolicy.py:289
      if (!finite_t(vel)) atomicOr(&s_bad_v, 1);
      if (!finite_t(nxt)) atomicCAS(&s_bad, -1, step);
      s_vals[i] = nxt;
    }
    __syncthreads();
    if (s_bad >= 0) break;  // the reference raises at the first bad step
  }
  // no CTA may exit while a peer could still push into its SMEM
  cluster.sync();
  if (cluster.block_rank() == 0) {
    for (int i = threadIdx.x; i < HD; i += blockDim.x) p.out_chunk[i] = s_vals[i];
    if (threadIdx.x == 0 && p.status) {
      p.status[0] = s_bad;
      p.status[1] = s_bad_v;
    }
  }
}

// ------------------------------------------------------- field evaluation

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
  int* status;
  int buf_elems, extra_elems;
};

// Field protocol evaluation (flowpolicy.py:203-209): v = (net([x,tau,emb,s]) - x)/(1 - tau).
template <typename T>
__global__ void __launch_bounds__(kThreads, 1) tiny_field_eval_kernel(const EvalParams<T> p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const Frame<T> f = frame<T>(smem_raw, p.buf_elems, p.extra_elems);
  prologue<T>(cluster, f, p.field, nullptr);
  const int n_in = p.field.sizes[0];
  for (int idx = threadIdx.x; idx < p.R * n_in; idx += blockDim.x) {
    const int r = idx / n_in, i = idx - r * n_in;
    T v;
    if (i < p.HD) v = p.x[r * p.HD + i];
    else if (i == p.HD) v = p.taus[r];
    else if (i < p.HD + 1 + p.emb_dim) v = p.emb[i - p.HD - 1];
    else v = p.state[i - p.HD - 1 - p.emb_dim];
    f.buf(0)[idx] = v;
  }
  __syncthreads();
  cluster.sync();  // every CTA's barriers are initialised before the first push
  uint32_t ph = 0;
  const T* out = f.buf(cluster_mlp<T>(cluster, f, p.field, f.bars0, p.R, f.buf(0), 1, 0, ph));
  cluster.sync();  // no CTA exits while its pushes to peers may be in flight
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

// ------------------------------------------------------------ MLP forward

template <typename T>
struct FwdParams {
  DevMlp<T> net;
  const T* x;
  int R;
  T* out;
  int buf_elems, extra_elems;
};

template <typename T>
__global__ void __launch_bounds__(kThreads, 1) tiny_mlp_forward_kernel(const FwdParams<T> p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const Frame<T> f = frame<T>(smem_raw, p.buf_elems, p.extra_elems);
  prologue<T>(cluster, f, p.net, nullptr);
  const int n_in = p.net.sizes[0], n_out = p.net.sizes[p.net.n_layers];
  for (int i = threadIdx.x; i < p.R * n_in; i += blockDim.x) f.buf(0)[i] = p.x[i];
  __syncthreads();
  cluster.sync();  // every CTA's barriers are initialised before the first push
  uint32_t ph = 0;
  const T* o = f.buf(cluster_mlp<T>(cluster, f, p.net, f.bars0, p.R, f.buf(0), 1, 0, ph));
  cluster.sync();  // no CTA exits while its pushes to peers may be in flight
  if (cluster.block_rank() == 0)
    for (int i = threadIdx.x; i < p.R * n_out; i += blockDim.x) p.out[i] = o[i];
}

// ------------------------------------------------------------- host side

int check_mlp(const sf_mlp_t* m, const char* name, size_t elem) {
  SF_REQUIRE(m->n_layers >= 1 && m->n_layers <= SF_MAX_LAYERS, "%s: bad layer count %d", name,
             m->n_layers);
  for (int i = 0; i < m->n_layers; ++i) {
    SF_REQUIRE(m->w[i] && m->b[i], "%s: null weights in layer %d", name, i);
    SF_REQUIRE(m->sizes[i] > 0 && m->sizes[i + 1] > 0, "%s: bad sizes", name);
    const int ld = m->ld[i] > 0 ? m->ld[i] : m->sizes[i];
    SF_REQUIRE(ld >= m->sizes[i], "%s: ld < n_in in layer %d", name, i);
    (void)elem;
  }
  return SF_OK;
}

int max_width(const sf_mlp_t* m) {
  int w = 0;
  for (int i = 0; m && i <= m->n_layers; ++i) w = w > m->sizes[i] ? w : m->sizes[i];
  return w;
}

// Assign SMEM arena slots to layers in execution order while they fit.
template <typename T>
size_t plan_arena(DevMlp<T>* first, DevMlp<T>* second, size_t fixed, int csize) {
  size_t off = 0;  // elements
  DevMlp<T>* order[2] = {first, second};
  for (DevMlp<T>* m : order) {
    if (!m) continue;
    for (int l = 0; l < m->n_layers; ++l) {
      m->woff[l] = -1;
      const size_t row_bytes = (size_t)m->ld[l] * sizeof(T);
      const uintptr_t base = reinterpret_cast<uintptr_t>(m->w[l]);
      if (row_bytes % 16 != 0 || base % 16 != 0) continue;  // bulk copies need 16 B granules
      const int rpc = (m->sizes[l + 1] + csize - 1) / csize;
      const size_t elems = (size_t)rpc * m->ld[l];
      if (fixed + (off + elems) * sizeof(T) > kSmemBudget) continue;
      m->woff[l] = (int)off;
      off += (elems + 15) & ~size_t(15);
    }
  }
  return fixed + off * sizeof(T);
}

int g_cluster16 = -1;  // 1 if 16-CTA clusters are schedulable, 0 if not, -1 unknown

// Per-kernel attribute cache: cudaFuncSetAttribute costs microseconds of host
// time, which would otherwise sit on the launch path of a ~10 us round.
template <typename K>
int ensure_attrs(K kern, size_t smem, int csize) {
  static size_t max_smem = 0;
  static bool nonportable = false;
  if (smem > max_smem) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kSmemBudget));
    max_smem = kSmemBudget;
  }
  if (csize > 8 && !nonportable) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    nonportable = true;
  }
  return SF_OK;
}

template <typename K>
int launch_cluster(K kern, const void* params_ptr, size_t smem, cudaStream_t stream, int csize) {
  int rc = ensure_attrs(kern, smem, csize);
  if (rc) return rc;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<void*>(params_ptr)};
  SF_CHECK_CUDA(cudaLaunchKernelExC(&cfg, (const void*)kern, args));
  count_launch();
  return SF_OK;
}

template <typename K>
int pick_cluster(K kern, size_t smem16) {
  if (g_cluster16 < 0) {
    g_cluster16 = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
            cudaSuccess &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem16) ==
            cudaSuccess) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem16;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 16;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &cfg) == cudaSuccess && n > 0)
        g_cluster16 = 1;
    }
    cudaGetLastError();
  }
  return g_cluster16 ? 16 : 8;
}

// Plan SMEM + cluster size, then launch.
template <typename T, typename P, typename K>
int plan_and_launch(K kern, P& p, DevMlp<T>* first, DevMlp<T>* second, int buf_elems,
                    int extra_elems, cudaStream_t stream) {
  p.buf_elems = (buf_elems + 15) & ~15;
  p.extra_elems = (extra_elems + 15) & ~15;
  const size_t fixed = frame_bytes<T>(p.buf_elems, p.extra_elems);
  SF_REQUIRE(fixed + 4096 <= kSmemBudget, "activation buffers need %zu B of shared memory", fixed);
  size_t smem = plan_arena<T>(first, second, fixed, 16);
  const int csize = pick_cluster(kern, smem);
  if (csize != 16) smem = plan_arena<T>(first, second, fixed, csize);
  return launch_cluster(kern, &p, smem, stream, csize);
}

template <typename T>
int flash_round_impl(const sf_mlp_t* draft_net, const void* draft_in, const sf_mlp_t* field_net,
                     const void* emb, int emb_dim, const void* state, int state_dim,
                     const void* eps, int H, int D, int C, const sf_verify_cfg_t* cfg,
                     const sf_verify_out_t* out, cudaStream_t stream) {
  FlashParams<T> p{};
  SF_REQUIRE(cfg, "null verifier config");
  SF_REQUIRE(cfg->k >= 1 && cfg->k <= kMaxRows, "tiny path supports 1..%d timesteps", kMaxRows);
  for (int i = 0; i < cfg->k; ++i) {
    SF_REQUIRE(cfg->taus[i] > 0.0 && cfg->taus[i] < 1.0,
               "verification timesteps must lie strictly inside (0, 1)");
    if (i) SF_REQUIRE(cfg->taus[i] > cfg->taus[i - 1], "verification timesteps must be strictly increasing");
    p.taus[i] = (T)cfg->taus[i];
  }
  SF_REQUIRE(cfg->delta >= 0.0, "delta must be non-negative");
  SF_REQUIRE(cfg->metric == SF_METRIC_L2 || cfg->metric == SF_METRIC_LINF, "unknown metric");
  SF_REQUIRE(cfg->current_sign == 1.0 || cfg->current_sign == -1.0,
             "current_sign must be -1.0 or +1.0");
  SF_REQUIRE(cfg->replan_size >= 1, "replan_size must be >= 1");
  SF_REQUIRE(field_net && draft_in && eps && out && out->branch_prefixes && out->result,
             "null argument");
  int rc;
  if ((rc = check_mlp(field_net, "field", sizeof(T)))) return rc;
  SF_REQUIRE(H >= 1 && D >= 2 && C >= 1 && C <= D - 1, "bad chunk shape H=%d D=%d C=%d", H, D, C);
  SF_REQUIRE(field_net->sizes[0] == H * D + 1 + emb_dim + state_dim,
             "velocity net dimensions do not match (H, D, emb, state)");
  SF_REQUIRE(field_net->sizes[field_net->n_layers] == H * D, "field output must be H*D");
  if (draft_net) {
    if ((rc = check_mlp(draft_net, "draft", sizeof(T)))) return rc;
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
  int width = max_width(field_net);
  if (draft_net) width = width > max_width(draft_net) ? width : max_width(draft_net);
  int buf = width * cfg->k;
  const int epi = cfg->k * H * D + cfg->k * H;  // recon + dist reuse a ping-pong buffer
  buf = buf > epi ? buf : epi;
  // weights of the net that runs first (draft) get SMEM first
  return plan_and_launch<T>(tiny_flash_round_kernel<T>, p, draft_net ? &p.draft : &p.field,
                            draft_net ? &p.field : nullptr, buf, H * D, stream);
}

template <typename T>
int full_round_impl(const sf_mlp_t* enc, const void* enc_in, int emb_dim, const sf_mlp_t* field_net,
                    const void* state, int state_dim, const void* start, int H, int D, int N,
                    void* chunk_out, void* emb_out, int* status, cudaStream_t stream) {
  int rc;
  SF_REQUIRE(enc_in && start && chunk_out, "null argument");
  SF_REQUIRE(N >= 0, "num_steps must be >= 0");
  SF_REQUIRE(field_net || N == 0, "null field");
  if (field_net && (rc = check_mlp(field_net, "field", sizeof(T)))) return rc;
  if (enc) {
    if ((rc = check_mlp(enc, "encoder", sizeof(T)))) return rc;
    SF_REQUIRE(enc->sizes[0] + enc->sizes[enc->n_layers] == emb_dim,
               "encoder embed_dim (in + out) must equal emb_dim");
  }
  if (field_net) {
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
  p.has_field = field_net != nullptr;
  p.state = static_cast<const T*>(state);
  p.state_dim = state_dim;
  p.start = static_cast<const T*>(start);
  p.H = H;
  p.D = D;
  p.N = field_net ? N : 0;
  p.out_chunk = static_cast<T*>(chunk_out);
  p.out_emb = static_cast<T*>(emb_out);
  p.status = status;
  int width = max_width(field_net);
  if (enc) width = width > max_width(enc) ? width : max_width(enc);
  // the field is reused N times: its weights get SMEM first
  DevMlp<T>* first = field_net ? &p.field : &p.enc;
  DevMlp<T>* second = (field_net && enc) ? &p.enc : nullptr;
  return plan_and_launch<T>(tiny_full_round_kernel<T>, p, first, second, width,
                            emb_dim + H * D + state_dim, stream);
}

template <typename T>
int field_eval_impl(const sf_mlp_t* field_net, const void* x, const double* taus, int R,
                    const void* emb, int emb_dim, const void* state, int state_dim, int H, int D,
                    void* out_v, int* status, cudaStream_t stream) {
  int rc;
  SF_REQUIRE(field_net && x && taus && out_v, "null argument");
  SF_REQUIRE(R >= 1 && R <= kMaxRows, "field evaluation supports 1..%d rows", kMaxRows);
  if ((rc = check_mlp(field_net, "field", sizeof(T)))) return rc;
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
  return plan_and_launch<T>(tiny_field_eval_kernel<T>, p, &p.field, nullptr,
                            max_width(field_net) * R, 0, stream);
}

template <typename T>
int mlp_forward_impl(const sf_mlp_t* net, const void* x, int R, void* out, cudaStream_t stream) {
  int rc;
  SF_REQUIRE(net && x && out, "null argument");
  SF_REQUIRE(R >= 1 && R <= kMaxRows, "mlp forward supports 1..%d rows", kMaxRows);
  if ((rc = check_mlp(net, "mlp", sizeof(T)))) return rc;
  FwdParams<T> p{};
  p.net = to_dev<T>(net);
  p.x = static_cast<const T*>(x);
  p.R = R;
  p.out = static_cast<T*>(out);
  return plan_and_launch<T>(tiny_mlp_forward_kernel<T>, p, &p.net, nullptr, max_width(net) * R, 0,
                            stream);
}

}  // namespace
}  // namespace sf

extern "C" int sf_tiny_flash_round(int precision, const sf_mlp_t* draft_net, const void* draft_in,
                                   const sf_mlp_t* field_net, const void* emb, int emb_dim,
                                   const void* state, int state_dim, const void* eps, int horizon,
                                   int dim, int continuous_dims, const sf_verify_cfg_t* cfg,
                                   const sf_verify_out_t* out, void* stream) {
  return SF_DISPATCH(precision, sf::flash_round_impl, draft_net, draft_in, field_net, emb, emb_dim,
                     state, state_dim, eps, horizon, dim, continuous_dims, cfg, out,
                     (cudaStream_t)stream);
}

// trace of the next tiny flash rounds (rank 0 stamps): on != 0 enables, out
// (32 u64) receives the stamps of the last round
extern "C" int sf_tiny_trace(int on, unsigned long long* out) {
  SF_CHECK_CUDA(cudaMemcpyToSymbol(sf::g_tiny_trace_on, &on, sizeof(int)));
  if (out) {
    SF_CHECK_CUDA(cudaDeviceSynchronize());
    SF_CHECK_CUDA(cudaMemcpyFromSymbol(out, sf::g_tiny_trace, 32 * sizeof(unsigned long long)));
  }
  return SF_OK;
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

extern "C" int sf_tiny_field_eval(int precision, const sf_mlp_t* field_net, const void* x,
                                  const double* taus, int rows, const void* emb, int emb_dim,
                                  const void* state, int state_dim, int horizon, int dim,
                                  void* velocity_out, int* status, void* stream) {
  return SF_DISPATCH(precision, sf::field_eval_impl, field_net, x, taus, rows, emb, emb_dim, state,
                     state_dim, horizon, dim, velocity_out, status, (cudaStream_t)stream);
}

extern "C" int sf_tiny_mlp_forward(int precision, const sf_mlp_t* net, const void* x, int rows,
                                   void* out, void* stream) {
  return SF_DISPATCH(precision, sf::mlp_forward_impl, net, x, rows, out, (cudaStream_t)stream);
}
