// Field-agnostic verification pieces (any field evaluated elsewhere):
// interpolation, verify epilogue, prefix scan, distances, gripper gate, Euler
// update. Reference: verifier.py:65-150, actions.py:168-211,
// flowpolicy.py:286-291.

#include <cuda_runtime.h>

#include "common.cuh"
#include "replan.cuh"
#include "verify_epi.cuh"

namespace sf {
namespace {

constexpr int kThreads = 256;

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

template <typename T>
__global__ void prefix_kernel(const T* d, int rows, int h, T delta, int* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= rows) return;
  const T* row = d + (size_t)warp * h;
  const int pre = warp_prefix<T>(h, delta, [&](int i) { return row[i]; });
  if ((threadIdx.x & 31) == 0) out[warp] = pre;
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
int load_cfg(const sf_verify_cfg_t* cfg, T* taus) {
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
  return SF_OK;
}

template <typename T>
int epilogue_impl(const void* draft, const void* eps, const void* vel, int H, int D, int C,
                  const sf_verify_cfg_t* cfg, const sf_verify_out_t* out, cudaStream_t stream) {
  EpiParams<T> p{};
  int rc = load_cfg<T>(cfg, p.taus);
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
  const int warps = 256 / 32;
  prefix_kernel<T><<<(rows + warps - 1) / warps, 256, 0, stream>>>(static_cast<const T*>(d), rows,
                                                                    h, (T)delta, out);
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

// ---- batched replanning bookkeeping (runtime.py:238-320), one CTA (replan.cuh)
__global__ void __launch_bounds__(1024) replan_update_kernel(int n, const int* __restrict__ result,
                                                             int* fsr, int* has_cache, int mode_flash,
                                                             int pf, int r, int* path, int* planned,
                                                             int* fb_idx, int* fb_count) {
  const int cnt = replan_update_cta(n, result, fsr, has_cache, mode_flash, pf, r, path, planned, fb_idx);
  if (threadIdx.x == 0) *fb_count = cnt;
}

}  // namespace
}  // namespace sf

extern "C" int sf_replan_update(int n_envs, const int* result, int* fsr, int* has_cache,
                                int mode_flash, int periodic_refresh, int replan_size, int* path,
                                int* planned, int* fb_idx, int* fb_count, void* stream) {
  SF_REQUIRE(n_envs >= 1 && fsr && has_cache && path && planned && fb_idx && fb_count,
             "bad replan arguments");
  SF_REQUIRE(result || !mode_flash, "flash mode needs the round's result words");
  SF_REQUIRE(replan_size >= 1 && periodic_refresh >= 0, "bad replan policy");
  sf::replan_update_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
      n_envs, result, fsr, has_cache, mode_flash, periodic_refresh, replan_size, path, planned,
      fb_idx, fb_count);
  SF_CHECK_CUDA(cudaGetLastError());
  sf::count_launch();
  return SF_OK;
}

extern "C" int sf_verify_epilogue(int precision, const void* draft, const void* eps,
                                  const void* velocity, int horizon, int dim, int continuous_dims,
                                  const sf_verify_cfg_t* cfg, const sf_verify_out_t* out,
                                  void* stream) {
  return SF_DISPATCH(precision, sf::epilogue_impl, draft, eps, velocity, horizon, dim,
                     continuous_dims, cfg, out, (cudaStream_t)stream);
}
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
