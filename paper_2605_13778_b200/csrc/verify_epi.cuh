// Verification epilogue shared by every verify entry point (tiny fused round,
// field-agnostic epilogue, pi0-scale chain): interpolation, endpoint
// reconstruction, per-step distances, per-branch longest-consistent prefix
// (warp ballots), min over branches, gripper gate, fallback decision.
//
// Reference: verifier.py:65-150, actions.py:168-211, runtime.py:286-320.
#pragma once

#include "common.cuh"

namespace sf {

// Decision for one env (runtime.py:286-320); writes result words.
__device__ __forceinline__ void write_decision(int L, int sw, int H, int phase_fallback,
                                               int prefix_cap, int replan_size, int nonfinite,
                                               int* out_result) {
  const bool phase_fb = phase_fallback && sw;
  const bool rejected = L == 0;
  int path, planned;
  if (phase_fb || rejected) {
    path = phase_fb ? SF_PATH_FLASH_PHASE : SF_PATH_FLASH_REJECTED;
    planned = replan_size;
  } else {
    path = SF_PATH_FLASH_ACCEPTED;
    planned = min(L, prefix_cap ? replan_size : H);
  }
  out_result[SF_RES_PREFIX] = L;
  out_result[SF_RES_SWITCH] = sw;
  out_result[SF_RES_PATH] = path;
  out_result[SF_RES_PLANNED] = planned;
  out_result[SF_RES_NONFINITE] = nonfinite;
}

// Longest leading run of d <= delta for one distance row, scanned by one warp
// with ballots (verifier.py:94-106). Comparison is inclusive and a NaN breaks
// the run (!(d <= delta)).
template <typename T, typename Get>
__device__ __forceinline__ int warp_prefix(int H, T delta, Get&& d) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < H; base += 32) {
    const int h = base + lane;
    const unsigned m = __ballot_sync(0xffffffffu, h < H && !(d(h) <= delta));
    if (m) return base + __ffs(m) - 1;
  }
  return H;
}

// One CTA verifies one env: `net_out(k, i)` yields the field output for
// branch k, element i (an endpoint when kEndpoint, else a velocity).
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
    const T x = add_rn(mul_rn(tau, draft[i]), mul_rn(omt, eps[i]));  // verifier.py:73
    const T v = kEndpoint ? div_rn(sub_rn(net_out(k, i), x), omt)     // flowpolicy.py:209
                          : net_out(k, i);
    const T recon = add_rn(x, mul_rn(omt, v));                          // verifier.py:88
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
  const int win = window < 0 ? H : (window < H ? window : H);
  for (int idx = threadIdx.x; idx < (K + 1) * win; idx += blockDim.x) {
    const int c = idx / win, h = idx - c * win;
    const T g = c == 0 ? draft[h * D + D - 1] : s_recon[(size_t)(c - 1) * HD + h * D + D - 1];
    if (mul_rn(g, sign) <= T(0)) s_switch = 1;  // actions.py:211; all writers store 1
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < K; k += blockDim.x >> 5) {
    const int pre = warp_prefix<T>(H, delta, [&](int h) { return s_dist[k * H + h]; });
    if (lane == 0) s_branch[k] = pre;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int L = H;
    for (int k = 0; k < K; ++k) {
      L = min(L, s_branch[k]);  // verifier.py:147
      out_branch[k] = s_branch[k];
    }
    write_decision(L, s_switch, H, phase_fallback, prefix_cap, replan_size,
                   s_nonfinite == 0x7fffffff ? -1 : s_nonfinite, out_result);
  }
}

}  // namespace sf
