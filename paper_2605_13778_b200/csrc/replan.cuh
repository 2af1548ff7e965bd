// Device-side round bookkeeping of a batch of independent envs (run_episode,
// runtime.py:238-320), shared by sf_replan_update (verify_ops.cu) and the
// graph-resident replanning round sf_ae_replan_round (pi0.cu).
#pragma once

#include "common.cuh"

namespace sf {

// One CTA (blockDim a multiple of 32, <= 1024):
//   forced = PF > 0 && fsr[e] >= PF; use_flash = mode_flash && has_cache[e] && !forced
//   !use_flash -> path FULL (PERIODIC if forced in flash mode), planned = R
//   flash      -> path / planned from the attempt's result words (planned = R on fallback)
//   fsr[e] += 1 on accepted rounds; every full round resets it and sets has_cache
// Envs that need the full (Euler) path are compacted in env order into
// fb_idx[0 .. count) by a block scan (deterministic); returns count on thread 0.
__device__ __forceinline__ int replan_update_cta(int n, const int* __restrict__ result, int* fsr,
                                                 int* has_cache, int mode_flash, int pf, int r,
                                                 int* path, int* planned, int* fb_idx) {
  __shared__ int warp_tot[32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int e = c0 + tid;
    int need = 0;
    if (e < n) {
      const int f = fsr[e];
      const bool forced = pf > 0 && f >= pf;
      const bool use_flash = mode_flash && has_cache[e] && !forced;
      int pth, pl;
      if (!use_flash) {
        pth = (forced && mode_flash) ? SF_PATH_PERIODIC : SF_PATH_FULL;
        pl = r;
      } else {
        pth = result[e * SF_RESULT_WORDS + SF_RES_PATH];
        pl = pth == SF_PATH_FLASH_ACCEPTED ? result[e * SF_RESULT_WORDS + SF_RES_PLANNED] : r;
      }
      need = pth != SF_PATH_FLASH_ACCEPTED;
      fsr[e] = need ? 0 : f + 1;
      if (need) has_cache[e] = 1;
      path[e] = pth;
      planned[e] = pl;
    }
    // block-wide exclusive scan of `need` (env order preserved)
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
      int v = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      warp_tot[lane] = v;  // inclusive
    }
    __syncthreads();
    const int before = (warp ? warp_tot[warp - 1] : 0) + __popc(m & ((1u << lane) - 1));
    if (need) fb_idx[base + before] = e;
    __syncthreads();
    if (tid == 0) base += warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  return base;
}

}  // namespace sf
