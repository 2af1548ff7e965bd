// MQA attention of the Action Expert's suffix tokens against the shared VLM
// prefix KV cache + the branch's own suffix keys (sm_100a, tcgen05 + TMA).
//
// Query rows are (token, head) pairs: row = token * 8 + head, so the Q
// activations [M, 8*256] are a contiguous [M*8, 256] K-major matrix and one
// 128-row tile = 16 tokens x 8 heads. All 8 heads share the single KV head
// (MQA), so every query tile multiplies the SAME 64-key K/V blocks:
//   S = Q K^T   (UMMA 128 x 64 x 256, fp32 in TMEM, double-buffered)
//   online softmax in registers (one thread per query row, exp2 with the
//   1/sqrt(d) scale folded in, lazy rescale when the row max grows by > 2^8)
//   O += P V    (UMMA 128 x 256 x 64; P bf16 via SMEM, V^T K-major from TMA)
// Keys = the env's P prefix keys (13 blocks of 64) + 2 blocks covering the
// suffix tokens of the (at most two) branch segments the tile touches, with
// the paper's block mask: the state token sees the
// prefix and itself, action tokens see the prefix and their branch's whole
// suffix. Batch-1 rounds split the key blocks across CTAs (split-KV) and the
// last CTA of each tile merges the partials in a fixed order.
#pragma once

#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "sm100.cuh"

namespace sf {
namespace attn {

namespace cg = cooperative_groups;

constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 softmax (2 per lane quarter)
constexpr int BQ = 128;     // query rows per tile (16 tokens x 8 heads)
constexpr int BKEY = 64;    // keys per block
constexpr int HD = 256;     // head dim
constexpr int kHeads = 8;
constexpr uint32_t kQBytes = BQ * HD * 2;         // 64 KB
constexpr uint32_t kKBytes = BKEY * HD * 2;       // 32 KB (4 chunks of 64 x 64)
constexpr uint32_t kVBytes = HD * BKEY * 2;       // 32 KB (V^T: 256 x 64)
constexpr uint32_t kPBytes = BQ * BKEY * 2;       // 16 KB
constexpr uint32_t kStageBytes = kKBytes + kVBytes;
// control region after P: mbarriers (256 B) + the softmax pair exchange (2 KB)
constexpr uint32_t kCtlBytes = 4096;
constexpr uint32_t kSmemBytes = kQBytes + 2 * kStageBytes + kPBytes + kCtlBytes + 1024 /*align*/;
constexpr int kTmemCols = 512;  // S0 [0,64) S1 [64,128) O [128,384) (+ P0/P1 bf16 [384,448))
// persistent kernel SMEM: Q | K slots | V^T slots (5 x 32 KB together) | barriers + row-max exchange (2 KB)
#ifndef SF_ATTN_KSLOTS
#define SF_ATTN_KSLOTS 2
#endif
constexpr int kPersistKSlots = SF_ATTN_KSLOTS;
constexpr int kPersistVSlots = 5 - SF_ATTN_KSLOTS;
constexpr uint32_t kPersistSmemUsed =
    kQBytes + kPersistKSlots * kKBytes + kPersistVSlots * kVBytes + 256 + 2 * 2 * BQ * 4;
constexpr uint32_t kPersistSmemBytes = 227 * 1024;  // the 1024 B alignment pad must fit in the slack
static_assert(kPersistSmemUsed <= kPersistSmemBytes, "persistent attention SMEM");
constexpr uint32_t kPCol = 384;  // persistent kernel: P(g) for slot s at kPCol + s * BKEY / 2
constexpr int kPartStride = HD + 2;  // split-KV partial O row stride in SMEM (floats)
constexpr int kMaxSplitsKV = 16;     // split-KV cluster size limit

struct Params {
  int M;            // valid token rows (n_envs * env_rows)
  int env_rows;     // rows per env: K * (1 + H), dense (no per-env padding)
  int n_envs;
  int tiles_env;    // 16-token query tiles per env: ceil(env_rows / 16); a
                    // tile never straddles two envs (one prefix per tile),
                    // rows past the env's last token are computed, not stored
  int seg_len;      // tokens per branch segment (1 + H)
  int segs;         // branches per env (K)
  int prefix_len;   // P
  int n_prefix_blocks;
  int n_blocks;     // n_prefix_blocks + suffix blocks
  int blocks_per_split;
  int splits;
  int tiles;
  float scale_log2;  // log2(e) / sqrt(HD)
  __nv_bfloat16* out;  // [M, 8*256]
  float* ws;           // [tiles][splits][128][HD + 2]
  int* counters;       // [tiles]
  const int* env_map;  // [envs] prefix-KV pool slot of each batch env (compacted batches)
  // prefix K / V^T as per-block SMEM images ([slot][block][32 KB], already
  // SWIZZLE_128B): one 32 KB bulk copy per operand instead of 4 + 1 tensor
  // boxes of 128 B rows (null: use the tensor maps)
  const uint8_t* k_img;
  const uint8_t* v_img;
  int img_blocks;      // key blocks per env image
  // optional live env count on the device (compacted bucket bodies of the
  // replanning graph): envs past it are not visited (batched kernels; null: n_envs)
  const int* envs_dev;
};

__device__ __forceinline__ int live_envs(const Params& p) {
  if (!p.envs_dev) return p.n_envs;
  const int n = __ldg(p.envs_dev);
  return n < p.n_envs ? n : p.n_envs;
}

#ifdef SF_TRACE
#define ATT_STAMP(i)                                                     \
  do {                                                                   \
    unsigned long long _t;                                               \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));               \
    stamps[i] = _t;                                                      \
  } while (0)
#else
#define ATT_STAMP(i) \
  do {               \
  } while (0)
#endif

// MUFU ex2 (flush-to-zero; ex2(-inf) = +0 for masked keys)
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// sm_100 three-input max
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float y;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(a), "f"(b), "f"(c));
  return y;
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// contiguous global -> shared bulk copy, completion counted on `bar` (bytes)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          sm100::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(sm100::smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* m, uint64_t* bar, void* dst, int c0,
                                            int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(sm100::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(sm100::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "l"(policy)
      : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kp,
                const __grid_constant__ CUtensorMap tm_vp, const __grid_constant__ CUtensorMap tm_ks,
                const __grid_constant__ CUtensorMap tm_vs, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + kQBytes;                      // 2 stages of [K 32KB | V 32KB]
  uint8_t* sP = sKV + 2 * kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kPBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [2] K half of a stage landed
  uint64_t* k_empty = bars + 3;   // [2] S(i) retired: K slot free
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* s_free = bars + 7;    // [2]
  uint64_t* p_full = bars + 9;    // [2]
  uint64_t* pv_done = bars + 11;  // [2]
  uint64_t* v_full = bars + 13;   // [2] V^T half landed
  uint64_t* v_empty = bars + 15;  // [2] PV(i) retired: V slot free
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  __shared__ unsigned long long stamps[16];
  (void)stamps;
#ifdef SF_TRACE
  __shared__ unsigned long long bt[6][16];  // per key block: kv_full, S commit, s_full seen, p arrive, PV commit, pv seen
#define BT(k, i)                                                  \
  do {                                                            \
    unsigned long long _t;                                        \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));        \
    if ((i) < 16) bt[k][i] = _t;                                  \
  } while (0)
#else
#define BT(k, i) \
  do {           \
  } while (0)
#endif
  if (threadIdx.x == 0) ATT_STAMP(0);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int env = tile / p.tiles_env;
  const int env_start = env * p.env_rows;
  const int m0 = env_start + (tile - env * p.tiles_env) * 16;  // first token of the tile
  const int seg_first = (m0 - env_start) / p.seg_len;
  // first suffix key token, rounded down to a 64-key boundary so every TMA box
  // of the transposed V starts on an aligned inner coordinate (3 blocks then
  // cover the <= 2 segments of 1 + H tokens the tile can touch)
  const int sb = (env_start + seg_first * p.seg_len) & ~(BKEY - 1);
  const int j0 = split * p.blocks_per_split;
  const int nb = min(p.blocks_per_split, p.n_blocks - j0);

  if (warp == 0 && lane == 0) {
    sm100::mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&k_full[s], 1);
      sm100::mbar_init(&k_empty[s], 1);
      sm100::mbar_init(&v_full[s], 1);
      sm100::mbar_init(&v_empty[s], 1);
      sm100::mbar_init(&s_full[s], 1);
      sm100::mbar_init(&s_free[s], 256);
    }
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&p_full[b], 256);
      sm100::mbar_init(&pv_done[b], 1);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) ATT_STAMP(1);
  float m_fin = -INFINITY, l_fin = 0.f;  // softmax rows' final (m, l) for the split-KV merge

  if (warp == 0) {
    if (sm100::elect_one()) {
      sm100::tma_prefetch_desc(&tm_q);
      sm100::tma_prefetch_desc(&tm_kp);
      sm100::tma_prefetch_desc(&tm_vp);
      sm100::tma_prefetch_desc(&tm_ks);
      sm100::tma_prefetch_desc(&tm_vs);
      const uint64_t pol_keep = sm100::policy_evict_last();
      const int slot = p.env_map ? __ldg(p.env_map + env) : env;  // prefix-KV pool slot
      // K and V^T halves of a key block are separate slots: K(i) reuses the
      // slot of K(i-2) once S(i-2) retired, V(i) the slot of V(i-2) once
      // PV(i-2) retired, so S(i) never waits behind the PV chain.
      auto load_k = [&](int i) {
        const int j = j0 + i;
        const int s = i & 1;
        uint8_t* st = sKV + s * kStageBytes;
        sm100::mbar_arrive_expect_tx(&k_full[s], kKBytes);
        if (j < p.n_prefix_blocks && p.k_img) {
          bulk_load(st, p.k_img + ((size_t)slot * p.img_blocks + j) * kKBytes, kKBytes, &k_full[s], pol_keep);
        } else if (j < p.n_prefix_blocks) {
          for (int c = 0; c < 4; ++c)
            tma_load_3d(&tm_kp, &k_full[s], st + c * (BKEY * 128), c * 64, j * BKEY, slot, pol_keep);
        } else {
          const int row0 = sb + (j - p.n_prefix_blocks) * BKEY;
          for (int c = 0; c < 4; ++c)
            sm100::tma_load_2d(&tm_ks, &k_full[s], st + c * (BKEY * 128), c * 64, row0, pol_keep);
        }
      };
      auto load_v = [&](int i) {
        const int j = j0 + i;
        const int s = i & 1;
        uint8_t* st = sKV + s * kStageBytes + kKBytes;
        sm100::mbar_arrive_expect_tx(&v_full[s], kVBytes);
        if (j < p.n_prefix_blocks && p.v_img) {
          bulk_load(st, p.v_img + ((size_t)slot * p.img_blocks + j) * kVBytes, kVBytes, &v_full[s], pol_keep);
        } else if (j < p.n_prefix_blocks) {
          tma_load_3d(&tm_vp, &v_full[s], st, j * BKEY, 0, slot, pol_keep);
        } else {
          const int row0 = sb + (j - p.n_prefix_blocks) * BKEY;
          sm100::tma_load_2d(&tm_vs, &v_full[s], st, row0, 0, pol_keep);
        }
      };
      // prefix K/V do not depend on the previous kernel: issue before the PDL wait
      int nk = 0, nv = 0;
      while (nk < min(2, nb) && j0 + nk < p.n_prefix_blocks) {
        load_k(nk);
        load_v(nk);
        ++nk;
        ++nv;
      }
      sm100::pdl_wait();
      sm100::mbar_arrive_expect_tx(q_full, kQBytes);
      for (int c = 0; c < 4; ++c)
        sm100::tma_load_2d(&tm_q, q_full, sQ + c * (BQ * 128), c * 64, m0 * kHeads, pol_keep);
      // two independent streams, issued in readiness order (polling)
      const long long t0 = clock64();
      while (nk < nb || nv < nb) {
        if (nk < nb && (nk < 2 || sm100::mbar_test(sm100::smem_u32(&k_empty[nk & 1]), ((nk >> 1) & 1) ^ 1))) {
          load_k(nk);
          ++nk;
        }
        if (nv < nb && nv < nk &&
            (nv < 2 || sm100::mbar_test(sm100::smem_u32(&v_empty[nv & 1]), ((nv >> 1) & 1) ^ 1))) {
          load_v(nv);
          ++nv;
        }
        if (clock64() - t0 > (1ll << 33)) {
          printf("sf: attention producer timeout (block %d)\n", blockIdx.x);
          __trap();
        }
      }
    }
  } else if (warp == 1) {
    if (sm100::elect_one()) {
      const uint32_t idesc_s = sm100::make_idesc_bf16(BQ, BKEY);
      const uint32_t idesc_o = sm100::make_idesc_bf16(BQ, HD);
      const uint32_t q_addr = sm100::smem_u32(sQ);
      const uint32_t p_addr = sm100::smem_u32(sP);
      sm100::mbar_wait(q_full, 0);
      ATT_STAMP(2);
      auto issue_pv = [&](int i) {
        sm100::mbar_wait(&p_full[i & 1], (i >> 1) & 1);
        sm100::tc_fence_after();
        sm100::mbar_wait(&v_full[i & 1], (i >> 1) & 1);
        sm100::tc_fence_after();
        const uint32_t v_addr = sm100::smem_u32(sKV + (i & 1) * kStageBytes + kKBytes);
        const uint32_t pb = p_addr;
#pragma unroll
        for (int kk = 0; kk < BKEY / 16; ++kk)
          sm100::umma_bf16(tmem + 128, sm100::make_sw128_desc(pb + kk * 32),
                           sm100::make_sw128_desc(v_addr + kk * 32), idesc_o, (i | kk) != 0);
        sm100::umma_commit(&pv_done[i & 1]);
        sm100::umma_commit(&v_empty[i & 1]);
        BT(4, i);
      };
      for (int i = 0; i < nb; ++i) {
        const int s = i & 1;
        sm100::mbar_wait(&k_full[s], (i >> 1) & 1);
        BT(0, i);
        if (i >= 2) sm100::mbar_wait(&s_free[s], ((i >> 1) & 1) ^ 1);
        sm100::tc_fence_after();
        const uint32_t k_addr = sm100::smem_u32(sKV + s * kStageBytes);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const int c = kk >> 2, w = kk & 3;
          sm100::umma_bf16(tmem + s * BKEY, sm100::make_sw128_desc(q_addr + c * (BQ * 128) + w * 32),
                           sm100::make_sw128_desc(k_addr + c * (BKEY * 128) + w * 32), idesc_s,
                           kk != 0);
        }
        sm100::umma_commit(&s_full[s]);
        sm100::umma_commit(&k_empty[s]);
        BT(1, i);
        if (i >= 1) issue_pv(i - 1);
      }
      if (nb > 0) issue_pv(nb - 1);
      ATT_STAMP(3);
    }
    __syncwarp();
  } else {
    // ------------------------------------------- softmax + correction + epilogue
    // Two warps per TMEM lane quarter (warps q+2 and q+6): each owns the same
    // 32 query rows and half of the columns (32 of a block's 64 keys; 128 of
    // O's 256 dims). The pair exchanges row maxima / sums through SMEM.
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = q * 32 + lane;  // query row in the tile == TMEM lane
    const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
    const int tok = m0 + (r >> 3);
    const int head = r & 7;
    const int local_q = tok - env_start;
    const int seg_q = local_q / p.seg_len;
    const int t_q = local_q - seg_q * p.seg_len;
    const bool real_q = local_q < p.segs * p.seg_len && tok < p.M;
    const bool store_q = local_q < p.env_rows && tok < p.M;  // the row's token belongs to this env
    const int seg_lo = seg_q * p.seg_len;                         // local token range of the
    const int seg_hi = seg_lo + (t_q >= 1 ? p.seg_len : 1);       // row's visible suffix keys
    __shared__ float xm[2 * 2 * BQ];                              // [2 parity][2 half][128]
    float m_used = -INFINITY, l_sum = 0.f;
    sm100::pdl_wait();
    if (threadIdx.x == 64) sm100::pdl_launch_dependents();
    for (int i = 0; i < nb; ++i) {
      const int j = j0 + i;
      const int s = i & 1;
      sm100::mbar_wait(&s_full[s], (i >> 1) & 1);
      if (threadIdx.x == 64) BT(2, i);
      sm100::tc_fence_after();
      uint32_t raw[2][16];
#pragma unroll
      for (int c = 0; c < 2; ++c) sm100::tmem_ld16(t_lane + s * BKEY + half * 32 + c * 16, raw[c]);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&s_free[s]);
      // valid keys of the row inside this block: [lo, hi) (block mask)
      int lo = 0, hi;
      if (j < p.n_prefix_blocks) {
        hi = p.prefix_len - j * BKEY;
      } else if (real_q) {
        const int base = sb + (j - p.n_prefix_blocks) * BKEY - env_start;  // local token of col 0
        lo = seg_lo - base;
        hi = seg_hi - base;
      } else {
        hi = 0;
      }
      lo -= half * 32;
      hi -= half * 32;
      float sv[32];
      float mb;
      if (lo <= 0 && hi >= 32) {  // fully visible half-block (every prefix block but the last)
#pragma unroll
        for (int c = 0; c < 32; ++c) sv[c] = __uint_as_float(raw[c >> 4][c & 15]);
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float x = __uint_as_float(raw[c >> 4][c & 15]);
          sv[c] = (c >= lo && c < hi) ? x : -INFINITY;
        }
      }
      {  // 3-input max tree
        float t[11];
#pragma unroll
        for (int c = 0; c < 10; ++c) t[c] = fmax3(sv[3 * c], sv[3 * c + 1], sv[3 * c + 2]);
        t[10] = fmaxf(sv[30], sv[31]);
        const float u0 = fmax3(t[0], t[1], t[2]), u1 = fmax3(t[3], t[4], t[5]);
        const float u2 = fmax3(t[6], t[7], t[8]), u3 = fmaxf(t[9], t[10]);
        mb = fmaxf(fmax3(u0, u1, u2), u3);
      }
      // pair max (raw scores; the positive scale commutes with max)
      xm[(s * 2 + half) * BQ + r] = mb;
      asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
      mb = fmaxf(xm[(s * 2) * BQ + r], xm[(s * 2 + 1) * BQ + r]) * p.scale_log2;
      const float m_new = fmaxf(m_used, mb);
      bool rescale = false;
      float alpha = 1.f;
      if (m_new > -INFINITY) {
        if (m_used == -INFINITY) {
          m_used = m_new;  // nothing accumulated yet: O and l are still zero
        } else if (m_new > m_used + 8.f) {
          alpha = exp2f(m_used - m_new);
          m_used = m_new;
          rescale = true;
        }
      }
      // P(i) overwrites P(i-1) and O may be rescaled: PV(i-1) must be done
      // (both warps of a pair decide the rescale alike)
      // exponentials first (registers): only the P store and an O rescale
      // have to wait for PV(i-1), so the MUFU work overlaps it
      const float mu = m_used == -INFINITY ? 0.f : m_used;
      uint32_t pw[16];
      float lp = 0.f;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float p0 = ex2_approx(fmaf(sv[2 * k], p.scale_log2, -mu));
        const float p1 = ex2_approx(fmaf(sv[2 * k + 1], p.scale_log2, -mu));
        lp += p0 + p1;
        __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
        pw[k] = *reinterpret_cast<uint32_t*>(&b2);
      }
      if (i >= 1) {
        sm100::mbar_wait(&pv_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
        if (threadIdx.x == 64) BT(5, i - 1);
        sm100::tc_fence_after();
      }
      const bool any_rescale = __any_sync(0xffffffffu, rescale);
      if (any_rescale && i >= 1) {
        l_sum *= alpha;
#pragma unroll 1
        for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 16) {
          uint32_t o[16];
          sm100::tmem_ld16(t_lane + 128 + c0, o);
          sm100::tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
          sm100::tmem_st16(t_lane + 128 + c0, o);
        }
        sm100::tmem_st_wait();
      } else if (rescale) {
        l_sum *= alpha;
      }
      // P row half (32 keys, bf16) into the SWIZZLE_128B K-major tile: 16 B
      // chunk c of row r lives at chunk (c ^ (r & 7)). p = 2^(x*scale - m).
      uint8_t* prow = sP + r * 128;
      l_sum += lp;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int cc = half * 4 + c;
        *reinterpret_cast<uint4*>(prow + ((cc ^ (r & 7)) << 4)) =
            make_uint4(pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
      }
      fence_async_smem();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&p_full[i & 1]);
      if (threadIdx.x == 64) BT(3, i);
    }
    // ---- epilogue: O row (256 fp32) is final once the last PV retires
    if (nb > 0) {
      sm100::mbar_wait(&pv_done[(nb - 1) & 1], ((nb - 1) >> 1) & 1);
      sm100::tc_fence_after();
    }
    // pair sum of l (each warp summed its own columns); the parity slot of
    // block nb was last read at block nb - 2, before the pair's last barrier
    {
      const int ps = nb & 1;
      xm[(ps * 2 + half) * BQ + r] = l_sum;
      asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
      l_sum = xm[(ps * 2) * BQ + r] + xm[(ps * 2 + 1) * BQ + r];
    }
    if (r == 0 && half == 0) ATT_STAMP(4);
    m_fin = m_used;
    l_fin = l_sum;
    if (p.splits == 1) {
      const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
      __nv_bfloat16* dst = p.out + (size_t)tok * (kHeads * HD) + head * HD;
      for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 32) {
        uint32_t o[2][16];
        sm100::tmem_ld16(t_lane + 128 + c0, o[0]);
        sm100::tmem_ld16(t_lane + 128 + c0 + 16, o[1]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          uint32_t w[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(o[u][2 * k]) * inv,
                                                      __uint_as_float(o[u][2 * k + 1]) * inv);
            w[k] = *reinterpret_cast<uint32_t*>(&b2);
          }
          if (store_q) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + c0 + 16 * u);
            d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
            d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
          }
        }
      }
    }
  }
  if (p.splits > 1) {
    // Split-KV merge over DSMEM (the S split CTAs of a tile are one cluster):
    // cluster rank t owns query rows [t*rows, t*rows + rows). After every
    // CTA's MMAs retired (cluster barrier 1: the K/V stage region is free),
    // each split pushes its unnormalised bf16 O rows and fp32 (m, l) straight
    // into the owner's SMEM ([split][HD/8 octets][rows] uint4, rows fastest:
    // conflict-free), cluster barrier 2 (release / acquire at cluster scope)
    // makes them visible, and the owner merges its rows from local SMEM in
    // a fixed split order (deterministic), accumulating in fp32. No L2
    // round trip for the partials.
    cg::cluster_group cluster = cg::this_cluster();
    const int S = p.splits;
    const int rows = (BQ + S - 1) / S;
    const int my_r0 = split * rows;
    const int my_nr = max(0, min(BQ, my_r0 + rows) - my_r0);
    uint4* recv_o = reinterpret_cast<uint4*>(sKV);                                  // [S][HD/8][rows]
    float2* recv_ml = reinterpret_cast<float2*>(sKV + (size_t)S * (HD / 8) * rows * 16);  // [S][rows]
    if (threadIdx.x == 64) ATT_STAMP(5);
    cluster.sync();  // every split's MMAs retired: the peers' K/V regions are free
    if (warp >= 2) {
      const int q = warp & 3;
      const int half = (warp - 2) >> 2;
      const int r = q * 32 + lane;
      const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
      const int owner = r / rows, rr = r - owner * rows;
      uint4* dst_o = cluster.map_shared_rank(recv_o, owner) + (size_t)split * (HD / 8) * rows + rr;
      if (half == 0)
        *(cluster.map_shared_rank(recv_ml, owner) + split * rows + rr) = make_float2(m_fin, l_fin);
#pragma unroll 1
      for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 64) {
        uint32_t o[4][16];
#pragma unroll
        for (int u = 0; u < 4; ++u) sm100::tmem_ld16(t_lane + 128 + c0 + 16 * u, o[u]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < 16; k += 8) {
            uint32_t w[4];
#pragma unroll
            for (int z = 0; z < 4; ++z) {
              __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(o[u][k + 2 * z]),
                                                        __uint_as_float(o[u][k + 2 * z + 1]));
              w[z] = *reinterpret_cast<uint32_t*>(&b2);
            }
            dst_o[(size_t)((c0 + 16 * u + k) >> 3) * rows] = make_uint4(w[0], w[1], w[2], w[3]);
          }
      }
    }
    cluster.sync();  // the partials of every split are in this CTA's SMEM
    if (threadIdx.x == 64) ATT_STAMP(6);
    // merge weights: wgt[row][s] = 2^(m_s - max_s m_s), inv[row] = 1 / sum_s wgt l_s
    float* wgt = reinterpret_cast<float*>(sP);  // [rows][S]
    float* inv = wgt + BQ * kMaxSplitsKV;       // [rows]
    if (threadIdx.x < my_nr) {
      float mx = -INFINITY;
      for (int s2 = 0; s2 < S; ++s2) mx = fmaxf(mx, recv_ml[s2 * rows + threadIdx.x].x);
      float L = 0.f;
      for (int s2 = 0; s2 < S; ++s2) {
        const float2 ml = recv_ml[s2 * rows + threadIdx.x];
        const float w = ml.x > -INFINITY ? exp2f(ml.x - mx) : 0.f;
        wgt[threadIdx.x * kMaxSplitsKV + s2] = w;
        L += w * ml.y;
      }
      inv[threadIdx.x] = L > 0.f ? 1.f / L : 0.f;
    }
    __syncthreads();
    const int total = my_nr * (HD / 8);
    for (int idx = threadIdx.x; idx < total; idx += kThreads) {
      const int rr = idx % my_nr, c8 = idx / my_nr;
      float a[8];
#pragma unroll
      for (int z = 0; z < 8; ++z) a[z] = 0.f;
      for (int s2 = 0; s2 < S; ++s2) {
        const uint4 v = recv_o[((size_t)s2 * (HD / 8) + c8) * rows + rr];
        const float w = wgt[rr * kMaxSplitsKV + s2];
        const uint32_t pk[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[z]));
          a[2 * z] += w * f.x;
          a[2 * z + 1] += w * f.y;
        }
      }
      const float iv = inv[rr];
      const int row = my_r0 + rr;
      const int tok = m0 + (row >> 3), head = row & 7;
      if (tok < p.M && tok - env_start < p.env_rows) {
        uint32_t w4[4];
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(a[2 * z] * iv, a[2 * z + 1] * iv);
          w4[z] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(p.out + (size_t)tok * (kHeads * HD) + head * HD + 8 * c8) =
            make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
    }
    if (threadIdx.x == 64) ATT_STAMP(7);
    if (threadIdx.x == 64) ATT_STAMP(8);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<kTmemCols>(tmem);
  }
#ifdef SF_TRACE
  if (threadIdx.x == 64 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && (blockIdx.y == 0 || blockIdx.y == gridDim.y - 1)) {
    ATT_STAMP(9);
    printf("attn trace blk(%d,%d) setup=%.2f q_ready=%.2f mma_done=%.2f pv_final=%.2f staged=%.2f csync1=%.2f merged=%.2f csync2=%.2f end=%.2f us\n",
           blockIdx.x, blockIdx.y, (stamps[1] - stamps[0]) * 1e-3, (stamps[2] - stamps[0]) * 1e-3,
           (stamps[3] - stamps[0]) * 1e-3, (stamps[4] - stamps[0]) * 1e-3, (stamps[5] - stamps[0]) * 1e-3,
           (stamps[6] - stamps[0]) * 1e-3, (stamps[7] - stamps[0]) * 1e-3, (stamps[8] - stamps[0]) * 1e-3,
           (stamps[9] - stamps[0]) * 1e-3);
    if (gridDim.y == 1)
      for (int i = 0; i < 16 && i < nb; ++i)
        printf("  blk %d: kv_full %.2f S_commit %.2f s_seen %.2f p_arrive %.2f PV_commit %.2f pv_seen %.2f\n", i,
               (bt[0][i] - stamps[0]) * 1e-3, (bt[1][i] - stamps[0]) * 1e-3, (bt[2][i] - stamps[0]) * 1e-3,
               (bt[3][i] - stamps[0]) * 1e-3, (bt[4][i] - stamps[0]) * 1e-3,
               i + 1 < nb ? (bt[5][i] - stamps[0]) * 1e-3 : -1.0);
  }
#endif
}

// ------------------------------------------------ batched: persistent
//
// attn_persistent_kernel (one KV split, batched rounds): one CTA per SM walks
// query tiles t = blockIdx.x, blockIdx.x + gridDim.x, ... with every barrier
// phase continuing across tiles (global key-block counter g = it * nb + i),
// so the NEXT tile's Q and first K/V blocks load while the current tile's
// last blocks and its epilogue run: Q is reloaded once the tile's last S MMA
// retired (q_empty), and PV(0) of the next tile (which overwrites O) waits for
// the softmax warps to have read O out of TMEM (o_free). Per block the
// pipeline is the attn_kernel one (separate K / V^T slots, 8 softmax warps).
__global__ void __launch_bounds__(kThreads, 1)
    attn_persistent_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kp,
                           const __grid_constant__ CUtensorMap tm_vp, const __grid_constant__ CUtensorMap tm_ks,
                           const __grid_constant__ CUtensorMap tm_vs, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kQBytes;               // kPersistKSlots x 32 KB
  uint8_t* sV = sK + kPersistKSlots * kKBytes;  // kPersistVSlots x 32 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kPersistVSlots * kVBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [<= 4]
  uint64_t* k_empty = bars + 5;   // [<= 4]
  uint64_t* s_full = bars + 9;    // [2]
  uint64_t* s_free = bars + 11;   // [2]
  uint64_t* p_full = bars + 13;   // [2]
  uint64_t* pv_done = bars + 15;  // [2]
  uint64_t* v_full = bars + 17;   // [<= 4]
  uint64_t* v_empty = bars + 21;  // [<= 4]
  uint64_t* q_empty = bars + 25;  // all S MMAs of a tile retired: Q reusable
  uint64_t* o_free = bars + 26;   // softmax warps read O out of TMEM: next PV(0) may overwrite
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 27);
  float* xm = reinterpret_cast<float*>(bars + 32);  // [2 slots][2 half][128]
  if (threadIdx.x == 0 && smem + kPersistSmemUsed > smem_raw + kPersistSmemBytes) __trap();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = p.envs_dev ? live_envs(p) * p.tiles_env : p.tiles;
  // tile -> first token, env, first suffix key block (sb) and the number of key
  // blocks the tile visits: the prefix blocks plus the suffix blocks covering
  // the segments of its 16 tokens (p.n_blocks is the bound over all tiles)
  auto tile_geom = [&](int tile, int& m0, int& env, int& env_start, int& sb, int& nbt) {
    env = tile / p.tiles_env;
    env_start = env * p.env_rows;
    m0 = env_start + (tile - env * p.tiles_env) * 16;
    const int lo = m0 - env_start;
    const int seg_first = lo / p.seg_len;
    int hi = min(lo + 15, p.segs * p.seg_len - 1);
    hi = hi < lo ? lo : hi;
    const int seg_last = hi / p.seg_len;
    sb = (env_start + seg_first * p.seg_len) & ~7;  // 8-key (16 B) aligned start of the tile's suffix keys
    const int n_suf = (env_start + (seg_last + 1) * p.seg_len - sb + BKEY - 1) / BKEY;
    nbt = p.n_prefix_blocks + min(n_suf, p.n_blocks - p.n_prefix_blocks);
  };

  if (warp == 0 && lane == 0) {
    sm100::mbar_init(q_full, 1);
    sm100::mbar_init(q_empty, 1);
    sm100::mbar_init(o_free, 256);
    for (int s = 0; s < kPersistKSlots; ++s) {
      sm100::mbar_init(&k_full[s], 1);
      sm100::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kPersistVSlots; ++s) {
      sm100::mbar_init(&v_full[s], 1);
      sm100::mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&s_full[s], 1);
      sm100::mbar_init(&s_free[s], 256);
      sm100::mbar_init(&p_full[s], 256);
      sm100::mbar_init(&pv_done[s], 1);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (sm100::elect_one()) {
      sm100::tma_prefetch_desc(&tm_q);
      sm100::tma_prefetch_desc(&tm_kp);
      sm100::tma_prefetch_desc(&tm_vp);
      sm100::tma_prefetch_desc(&tm_ks);
      sm100::tma_prefetch_desc(&tm_vs);
      const uint64_t pol = sm100::policy_evict_last();
      // Block cursors (tile it, key block j) for the next K and V loads, advanced
      // incrementally (no 64-bit divisions on the issuing thread); the tile's
      // prefix-KV pool slot and first suffix block are looked up once per tile.
      // K(g) reuses the slot of K(g-3) once S(g-3) retired, V(g) that of V(g-2)
      // once PV(g-2) retired.
      struct Cursor {
        int it = 0, j = 0, slot = 0, sb = 0, nb = 0;
      };
      auto cursor_tile = [&](Cursor& c) {
        const int tile = blockIdx.x + c.it * gridDim.x;
        if (tile >= n_tiles) return;  // past this CTA's last tile
        int m0, env, env_start;
        tile_geom(tile, m0, env, env_start, c.sb, c.nb);
        c.slot = p.env_map ? __ldg(p.env_map + env) : env;
      };
      auto cursor_next = [&](Cursor& c) {
        if (++c.j == c.nb) {
          c.j = 0;
          ++c.it;
          cursor_tile(c);
        }
      };
      Cursor ck, cv;
      cursor_tile(ck);
      cv = ck;
      int k_s = 0;
      uint32_t k_ph = 0;  // slot and ring phase of the next K
      auto load_k = [&]() {
        const int j = ck.j, slot = ck.slot, sb = ck.sb;
        const int s = k_s;
        uint8_t* st = sK + s * kKBytes;
        sm100::mbar_arrive_expect_tx(&k_full[s], kKBytes);
        if (j < p.n_prefix_blocks && p.k_img) {
          bulk_load(st, p.k_img + ((size_t)slot * p.img_blocks + j) * kKBytes, kKBytes, &k_full[s], pol);
        } else if (j < p.n_prefix_blocks) {
          for (int c = 0; c < 4; ++c)
            tma_load_3d(&tm_kp, &k_full[s], st + c * (BKEY * 128), c * 64, j * BKEY, slot, pol);
        } else {
          const int row0 = sb + (j - p.n_prefix_blocks) * BKEY;
          for (int c = 0; c < 4; ++c)
            sm100::tma_load_2d(&tm_ks, &k_full[s], st + c * (BKEY * 128), c * 64, row0, pol);
        }
        if (++k_s == kPersistKSlots) {
          k_s = 0;
          k_ph ^= 1;
        }
        cursor_next(ck);
      };
      int v_s = 0;
      uint32_t v_ph = 0;  // slot and ring phase of the next V
      auto load_v = [&]() {
        const int j = cv.j, slot = cv.slot, sb = cv.sb;
        const int s = v_s;
        uint8_t* st = sV + s * kVBytes;
        sm100::mbar_arrive_expect_tx(&v_full[s], kVBytes);
        if (j < p.n_prefix_blocks && p.v_img) {
          bulk_load(st, p.v_img + ((size_t)slot * p.img_blocks + j) * kVBytes, kVBytes, &v_full[s], pol);
        } else if (j < p.n_prefix_blocks) {
          tma_load_3d(&tm_vp, &v_full[s], st, j * BKEY, 0, slot, pol);
        } else {
          const int row0 = sb + (j - p.n_prefix_blocks) * BKEY;
          sm100::tma_load_2d(&tm_vs, &v_full[s], st, row0, 0, pol);
        }
        if (++v_s == kPersistVSlots) {
          v_s = 0;
          v_ph ^= 1;
        }
        cursor_next(cv);
      };
      const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      long long nk = 0, nv = 0;
      int nq = 0;  // Q tiles issued
      // prefix blocks of the first tile before the PDL wait (independent of the previous kernel)
      while (my_tiles > 0 && nk < 2 && (int)nk < p.n_prefix_blocks) {
        load_k();
        load_v();
        ++nk;
        ++nv;
      }
      sm100::pdl_wait();
      const long long t0 = clock64();
      while (ck.it < my_tiles || cv.it < my_tiles || nq < my_tiles) {
        // Q of tile nq once every S MMA of tile nq-1 retired
        if (nq < my_tiles && (nq == 0 || sm100::mbar_test(sm100::smem_u32(q_empty), (nq - 1) & 1))) {
          int m0, env, env_start, sb, nbt;
          tile_geom(blockIdx.x + nq * gridDim.x, m0, env, env_start, sb, nbt);
          sm100::mbar_arrive_expect_tx(q_full, kQBytes);
          for (int c = 0; c < 4; ++c)
            sm100::tma_load_2d(&tm_q, q_full, sQ + c * (BQ * 128), c * 64, m0 * kHeads, pol);
          ++nq;
        }
        if (ck.it < my_tiles && (nk < kPersistKSlots || sm100::mbar_test(sm100::smem_u32(&k_empty[k_s]), k_ph ^ 1))) {
          load_k();
          ++nk;
        }
        if (cv.it < my_tiles && nv < nk &&
            (nv < kPersistVSlots || sm100::mbar_test(sm100::smem_u32(&v_empty[v_s]), v_ph ^ 1))) {
          load_v();
          ++nv;
        }
        if (clock64() - t0 > (1ll << 34)) {
          printf("sf: attention producer timeout (block %d)\n", blockIdx.x);
          __trap();
        }
      }
    }
  } else if (warp == 1) {
    if (sm100::elect_one()) {
      const uint32_t idesc_s = sm100::make_idesc_bf16(BQ, BKEY);
      const uint32_t idesc_o = sm100::make_idesc_bf16(BQ, HD);
      const uint32_t q_addr = sm100::smem_u32(sQ);
      long long g = 0;
      int it = 0;
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;  // K ring slot / phase of block g, V ring of the next PV
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        const long long g0 = g;
        sm100::mbar_wait(q_full, it & 1);
        auto issue_pv = [&](long long gg) {
          const int i = (int)(gg - g0);
          if (i == 0 && it > 0) {  // PV(0) overwrites O: the previous tile's O must be drained
            sm100::mbar_wait(o_free, (it - 1) & 1);
          }
          sm100::mbar_wait(&p_full[gg & 1], (gg >> 1) & 1);
          sm100::mbar_wait(&v_full[vs], vph);
          sm100::tc_fence_after();
          const uint32_t v_addr = sm100::smem_u32(sV + vs * kVBytes);
          const uint32_t p_tmem = tmem + kPCol + (uint32_t)(gg & 1) * (BKEY / 2);
#pragma unroll
          for (int kk = 0; kk < BKEY / 16; ++kk)  // A = P from TMEM: 16 keys = 8 columns per MMA
            sm100::umma_bf16_ts(tmem + 128, p_tmem + kk * 8, sm100::make_sw128_desc(v_addr + kk * 32),
                                idesc_o, (i | kk) != 0);
          sm100::umma_commit(&pv_done[gg & 1]);
          sm100::umma_commit(&v_empty[vs]);
          if (++vs == kPersistVSlots) {
            vs = 0;
            vph ^= 1;
          }
        };
        int m0, env, env_start, sb, nb;
        tile_geom(tile, m0, env, env_start, sb, nb);
        for (int i = 0; i < nb; ++i, ++g) {
          const int s = (int)(g & 1);
          sm100::mbar_wait(&k_full[ks], kph);
          if (g >= 2) sm100::mbar_wait(&s_free[s], ((g >> 1) & 1) ^ 1);
          sm100::tc_fence_after();
          const uint32_t k_addr = sm100::smem_u32(sK + ks * kKBytes);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const int c = kk >> 2, w = kk & 3;
            sm100::umma_bf16(tmem + s * BKEY, sm100::make_sw128_desc(q_addr + c * (BQ * 128) + w * 32),
                             sm100::make_sw128_desc(k_addr + c * (BKEY * 128) + w * 32), idesc_s, kk != 0);
          }
          sm100::umma_commit(&s_full[s]);
          sm100::umma_commit(&k_empty[ks]);
          if (++ks == kPersistKSlots) {
            ks = 0;
            kph ^= 1;
          }
          if (i == nb - 1) sm100::umma_commit(q_empty);  // last S of the tile: Q reusable
          if (i >= 1) issue_pv(g - 1);
        }
        if (nb > 0) issue_pv(g - 1);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
    sm100::pdl_wait();
    if (threadIdx.x == 64) sm100::pdl_launch_dependents();
    long long g = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      int m0, env, env_start, sb, nb;
      tile_geom(tile, m0, env, env_start, sb, nb);
      const int tok = m0 + (r >> 3);
      const int head = r & 7;
      const int local_q = tok - env_start;
      const int seg_q = local_q / p.seg_len;
      const int t_q = local_q - seg_q * p.seg_len;
      const bool real_q = local_q < p.segs * p.seg_len && tok < p.M;
      const bool store_q = local_q < p.env_rows && tok < p.M;  // the row's token belongs to this env
      const int seg_lo = seg_q * p.seg_len;
      const int seg_hi = seg_lo + (t_q >= 1 ? p.seg_len : 1);
      float m_used = -INFINITY, l_sum = 0.f;
      for (int i = 0; i < nb; ++i, ++g) {
        const int j = i;
        const int s = (int)(g & 1);
        sm100::mbar_wait(&s_full[s], (g >> 1) & 1);
        sm100::tc_fence_after();
        uint32_t raw[2][16];
#pragma unroll
        for (int c = 0; c < 2; ++c) sm100::tmem_ld16(t_lane + s * BKEY + half * 32 + c * 16, raw[c]);
        sm100::tmem_ld_wait();
        sm100::tc_fence_before();
        sm100::mbar_arrive(&s_free[s]);
        int lo = 0, hi;
        if (j < p.n_prefix_blocks) {
          hi = p.prefix_len - j * BKEY;
        } else if (real_q) {
          const int base = sb + (j - p.n_prefix_blocks) * BKEY - env_start;
          lo = seg_lo - base;
          hi = seg_hi - base;
        } else {
          hi = 0;
        }
        lo -= half * 32;
        hi -= half * 32;
        float sv[32];
        float mb;
        if (lo <= 0 && hi >= 32) {
#pragma unroll
          for (int c = 0; c < 32; ++c) sv[c] = __uint_as_float(raw[c >> 4][c & 15]);
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float x = __uint_as_float(raw[c >> 4][c & 15]);
            sv[c] = (c >= lo && c < hi) ? x : -INFINITY;
          }
        }
        {
          float t[11];
#pragma unroll
          for (int c = 0; c < 10; ++c) t[c] = fmax3(sv[3 * c], sv[3 * c + 1], sv[3 * c + 2]);
          t[10] = fmaxf(sv[30], sv[31]);
          const float u0 = fmax3(t[0], t[1], t[2]), u1 = fmax3(t[3], t[4], t[5]);
          const float u2 = fmax3(t[6], t[7], t[8]), u3 = fmaxf(t[9], t[10]);
          mb = fmaxf(fmax3(u0, u1, u2), u3);
        }
        xm[(s * 2 + half) * BQ + r] = mb;
        asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
        mb = fmaxf(xm[(s * 2) * BQ + r], xm[(s * 2 + 1) * BQ + r]) * p.scale_log2;
        const float m_new = fmaxf(m_used, mb);
        bool rescale = false;
        float alpha = 1.f;
        if (m_new > -INFINITY) {
          if (m_used == -INFINITY) {
            m_used = m_new;
          } else if (m_new > m_used + 8.f) {
            alpha = exp2f(m_used - m_new);
            m_used = m_new;
            rescale = true;
          }
        }
        const float mu = m_used == -INFINITY ? 0.f : m_used;
        uint32_t pw[16];
        float lp = 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float p0 = ex2_approx(fmaf(sv[2 * k], p.scale_log2, -mu));
          const float p1 = ex2_approx(fmaf(sv[2 * k + 1], p.scale_log2, -mu));
          lp += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          pw[k] = *reinterpret_cast<uint32_t*>(&b2);
        }
        // P slot s is free once PV(g-2) retired; PV(g-1) may still run
        // unless O has to be rescaled
        if (g >= 2) {
          sm100::mbar_wait(&pv_done[s], ((g - 2) >> 1) & 1);
          sm100::tc_fence_after();
        }
        const bool any_rescale = __any_sync(0xffffffffu, rescale);
        if (any_rescale && i >= 1) {
          sm100::mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
          sm100::tc_fence_after();
          l_sum *= alpha;
#pragma unroll 1
          for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 16) {
            uint32_t o[16];
            sm100::tmem_ld16(t_lane + 128 + c0, o);
            sm100::tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
            sm100::tmem_st16(t_lane + 128 + c0, o);
          }
          sm100::tmem_st_wait();
        } else if (rescale) {
          l_sum *= alpha;
        }
        l_sum += lp;
        sm100::tmem_st16(t_lane + kPCol + s * (BKEY / 2) + half * 16, pw);
        sm100::tmem_st_wait();
        sm100::tc_fence_before();
        sm100::mbar_arrive(&p_full[s]);
      }
      // O final once the tile's last PV retires
      if (nb > 0) {
        sm100::mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
        sm100::tc_fence_after();
      }
      // row sums through slot g & 1 (last read for block g - 2, before block g - 1's barrier)
      const int ls = (int)(g & 1);
      xm[(ls * 2 + half) * BQ + r] = l_sum;
      asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
      l_sum = xm[(ls * 2) * BQ + r] + xm[(ls * 2 + 1) * BQ + r];
      asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");  // slot free for the next tile's block g
      const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
      // O -> registers first, then release TMEM (the next tile's PV(0) may
      // start), then the slow global stores
      uint32_t ow[4][2][8];
#pragma unroll
      for (int u4 = 0; u4 < 4; ++u4) {
        uint32_t o[2][16];
        const int c0 = half * 128 + u4 * 32;
        sm100::tmem_ld16(t_lane + 128 + c0, o[0]);
        sm100::tmem_ld16(t_lane + 128 + c0 + 16, o[1]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(o[u][2 * k]) * inv,
                                                      __uint_as_float(o[u][2 * k + 1]) * inv);
            ow[u4][u][k] = *reinterpret_cast<uint32_t*>(&b2);
          }
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive(o_free);
      if (store_q) {
        __nv_bfloat16* dst = p.out + (size_t)tok * (kHeads * HD) + head * HD + half * 128;
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4)
#pragma unroll
          for (int u = 0; u < 2; ++u)  // 16 dims = one full 32 B sector per store
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + u4 * 32 + 16 * u),
                         "r"(ow[u4][u][0]), "r"(ow[u4][u][1]), "r"(ow[u4][u][2]), "r"(ow[u4][u][3]),
                         "r"(ow[u4][u][4]), "r"(ow[u4][u][5]), "r"(ow[u4][u][6]), "r"(ow[u4][u][7])
                         : "memory");
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

// ------------------------------------------------ batched: 2-SM CTA pairs
//
// attn_pair_kernel (persistent, one KV split, batched rounds): the two CTAs
// of a cluster run two consecutive query tiles of one env ("pair tile", 32
// tokens x 8 heads = 256 query rows) with tcgen05.mma.cta_group::2 over
// 128-key superblocks (two 64-key blocks; CTA r loads block 2G + r):
//   S(G) = Q K^T   one 256 x 128 MMA group (N = 128 halves the number of S
//                  MMAs per key, the costliest part of the 1-SM kernel);
//                  each CTA holds its 128 query rows of S in TMEM;
//   P(G)           written by the softmax (bf16) over the first 64 columns of
//                  S(G)'s TMEM slot;
//   O += P V       one 256 x 256 MMA group with A = P from each CTA's TMEM and
//                  V^T split by dims (CTA r holds dims [128 r, 128 r + 128)).
// Per superblock each SM loads 32 KB of K and 32 KB of V^T (the 1-SM kernel
// loads 64 KB per 64 keys). S(G+2) reuses P(G)'s slot: it is issued after
// PV(G) and tcgen05 MMAs of one issuer execute in order. The leader (rank 0)
// issues every MMA; its full-barriers count both CTAs' TMA bytes
// (.cta_group::2 loads signal the leader), its p_full / o_free barriers one
// arrival per softmax warp of both CTAs; MMA commits are multicast. Pair
// tiles are walked persistently with barrier phases continuing across them;
// an odd last tile of an env gets a dummy partner whose rows are dropped.

constexpr int kPairKSlots = 2;
constexpr int kPairVSlots = 3;
constexpr uint32_t kPairKBytes = BKEY * HD * 2;        // 32 KB: this CTA's 64-key block (4 chunks of 64 x 64)
constexpr uint32_t kPairVBytes = (HD / 2) * 128 * 2;   // 32 KB: 128 dims x 128 keys (2 chunks of 128 x 64)
constexpr uint32_t kPairSmemUsed =
    kQBytes + kPairKSlots * kPairKBytes + kPairVSlots * kPairVBytes + 256 + 2 * 2 * BQ * 4;
constexpr uint32_t kPairSmemBytes = 227 * 1024;
static_assert(kPairSmemUsed <= kPairSmemBytes, "pair attention SMEM");
constexpr uint32_t kPairOCol = 256;  // TMEM: S/P slots [0,128) [128,256), O [256,512)

__device__ __forceinline__ uint32_t pair_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t pair_mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void pair_load_2d(const CUtensorMap* m, uint32_t bar, void* dst, int c0, int c1,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(sm100::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void pair_load_3d(const CUtensorMap* m, uint32_t bar, void* dst, int c0, int c1,
                                             int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(sm100::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void pair_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// A from each CTA's own TMEM (its 128 rows), B halves from the two SMEMs.
__device__ __forceinline__ void pair_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void pair_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          sm100::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// Remote (or local, via mapa) arrive with the default .release.cta semantics
// (the CUTLASS cluster-barrier form): the data it publishes lives in TMEM and
// is ordered by tcgen05 fences; a .release.cluster arrive would emit a
// GPU-scope MEMBAR per call.
__device__ __forceinline__ void pair_arrive(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kp,
                     const __grid_constant__ CUtensorMap tm_vp, const __grid_constant__ CUtensorMap tm_ks,
                     const __grid_constant__ CUtensorMap tm_vs, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kQBytes;                  // kPairKSlots x 32 KB
  uint8_t* sV = sK + kPairKSlots * kPairKBytes;  // kPairVSlots x 32 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kPairVSlots * kPairVBytes);
  uint64_t* q_full = bars + 0;    // leader: both Q tiles landed
  uint64_t* k_full = bars + 1;    // [2] leader: both K blocks landed
  uint64_t* k_empty = bars + 3;   // [2] both: S of the superblock retired
  uint64_t* s_full = bars + 5;    // [2] both
  uint64_t* p_full = bars + 7;    // [2] leader: both CTAs wrote P
  uint64_t* pv_done = bars + 9;   // [2] both
  uint64_t* v_full = bars + 11;   // [3] leader: both V^T halves landed
  uint64_t* v_empty = bars + 14;  // [3] both: PV of the superblock retired
  uint64_t* q_empty = bars + 17;  // both: every S of the pair tile retired
  uint64_t* o_free = bars + 18;   // leader: both CTAs drained O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 19);
  float* xm = reinterpret_cast<float*>(bars + 32);  // [2 slots][2 half][128]
  if (threadIdx.x == 0 && smem + kPairSmemUsed > smem_raw + kPairSmemBytes) __trap();
  cg::cluster_group cluster = cg::this_cluster();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = pair_rank();
  const bool leader = rank == 0;
  const int tiles_env = p.tiles_env;
  const int pairs_env = (tiles_env + 1) / 2;
  const int n_pairs = live_envs(p) * pairs_env;
  const int cl = blockIdx.x >> 1, n_cl = gridDim.x >> 1;
  const int my_pairs = cl < n_pairs ? (n_pairs - 1 - cl) / n_cl + 1 : 0;
  // pair tile -> env, this CTA's first token, validity, first suffix key block
  // and key-block count (prefix + suffix blocks covering the pair's segments)
  auto pair_geom = [&](int pt, int& env, int& env_start, int& m0, bool& valid, int& sb, int& nbt) {
    env = pt / pairs_env;
    const int jp = pt - env * pairs_env;
    env_start = env * p.env_rows;
    const int tloc = 2 * jp + (int)rank;
    valid = tloc < tiles_env;
    m0 = env_start + tloc * 16;
    const int lo = 32 * jp;
    const int seg_first = lo / p.seg_len;
    int hi = min(lo + 31, p.segs * p.seg_len - 1);
    hi = hi < lo ? lo : hi;
    const int seg_last = hi / p.seg_len;
    sb = (env_start + seg_first * p.seg_len) & ~7;  // 8-key (16 B) aligned: V^T boxes start on the key axis
    const int n_suf = (env_start + (seg_last + 1) * p.seg_len - sb + BKEY - 1) / BKEY;
    nbt = p.n_prefix_blocks + min(n_suf, p.n_blocks - p.n_prefix_blocks);
  };

  if (warp == 0 && lane == 0) {
    sm100::mbar_init(q_full, 1);
    sm100::mbar_init(q_empty, 1);
    sm100::mbar_init(o_free, 2 * 8);  // one arrival per softmax warp
    for (int s = 0; s < kPairKSlots; ++s) {
      sm100::mbar_init(&k_full[s], 1);
      sm100::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kPairVSlots; ++s) {
      sm100::mbar_init(&v_full[s], 1);
      sm100::mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&s_full[s], 1);
      sm100::mbar_init(&p_full[s], 2 * 8);
      sm100::mbar_init(&pv_done[s], 1);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        sm100::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  sm100::tc_fence_before();
  cluster.sync();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (sm100::elect_one()) {
      sm100::tma_prefetch_desc(&tm_q);
      sm100::tma_prefetch_desc(&tm_kp);
      sm100::tma_prefetch_desc(&tm_vp);
      sm100::tma_prefetch_desc(&tm_ks);
      sm100::tma_prefetch_desc(&tm_vs);
      const uint64_t pol = sm100::policy_evict_last();
      // superblock cursors (pair tile it, superblock G) for the next K and V loads
      struct Cursor {
        int it = 0, G = 0, slot = 0, sb = 0, nb = 0;
      };
      auto cursor_tile = [&](Cursor& c) {
        if (c.it >= my_pairs) return;
        int env, env_start, m0;
        bool valid;
        pair_geom(cl + c.it * n_cl, env, env_start, m0, valid, c.sb, c.nb);
        c.slot = p.env_map ? __ldg(p.env_map + env) : env;
      };
      auto cursor_next = [&](Cursor& c) {
        if (++c.G == (c.nb + 1) / 2) {
          c.G = 0;
          ++c.it;
          cursor_tile(c);
        }
      };
      Cursor ck, cv;
      cursor_tile(ck);
      cv = ck;
      int k_s = 0, v_s = 0;
      uint32_t k_ph = 0, v_ph = 0;
      // a block past the tile's last one (odd count) re-reads prefix block 0:
      // finite data, fully masked by the softmax
      auto load_k = [&]() {
        const int s = k_s;
        uint8_t* st = sK + s * kPairKBytes;
        const uint32_t fb = pair_mapa(sm100::smem_u32(&k_full[s]), 0);
        if (leader) sm100::mbar_arrive_expect_tx(&k_full[s], 2 * kPairKBytes);
        int j = 2 * ck.G + (int)rank;
        j = j < ck.nb ? j : 0;
        if (j < p.n_prefix_blocks) {
          for (int c = 0; c < 4; ++c)
            pair_load_3d(&tm_kp, fb, st + c * (BKEY * 128), c * 64, j * BKEY, ck.slot, pol);
        } else {
          const int row0 = ck.sb + (j - p.n_prefix_blocks) * BKEY;
          for (int c = 0; c < 4; ++c) pair_load_2d(&tm_ks, fb, st + c * (BKEY * 128), c * 64, row0, pol);
        }
        if (++k_s == kPairKSlots) {
          k_s = 0;
          k_ph ^= 1;
        }
        cursor_next(ck);
      };
      auto load_v = [&]() {
        const int s = v_s;
        uint8_t* st = sV + s * kPairVBytes;
        const uint32_t fb = pair_mapa(sm100::smem_u32(&v_full[s]), 0);
        if (leader) sm100::mbar_arrive_expect_tx(&v_full[s], 2 * kPairVBytes);
        for (int h = 0; h < 2; ++h) {  // chunk h: keys of block 2G + h, this CTA's 128 dims
          int j = 2 * cv.G + h;
          j = j < cv.nb ? j : 0;
          uint8_t* dst = st + h * (kPairVBytes / 2);
          if (j < p.n_prefix_blocks) {
            pair_load_3d(&tm_vp, fb, dst, j * BKEY, (int)rank * (HD / 2), cv.slot, pol);
          } else {
            const int row0 = cv.sb + (j - p.n_prefix_blocks) * BKEY;
            pair_load_2d(&tm_vs, fb, dst, row0, (int)rank * (HD / 2), pol);
          }
        }
        if (++v_s == kPairVSlots) {
          v_s = 0;
          v_ph ^= 1;
        }
        cursor_next(cv);
      };
      long long nk = 0, nv = 0;
      int nq = 0;
      const uint32_t qb = pair_mapa(sm100::smem_u32(q_full), 0);
      // prefix superblock 0 of the first pair tile before the PDL wait
      if (my_pairs > 0 && 2 <= p.n_prefix_blocks) {
        load_k();
        load_v();
        ++nk;
        ++nv;
      }
      sm100::pdl_wait();
      const long long t0 = clock64();
      while (ck.it < my_pairs || cv.it < my_pairs || nq < my_pairs) {
        if (nq < my_pairs && (nq == 0 || sm100::mbar_test(sm100::smem_u32(q_empty), (nq - 1) & 1))) {
          int env, env_start, m0, sb, nbt;
          bool valid;
          pair_geom(cl + nq * n_cl, env, env_start, m0, valid, sb, nbt);
          if (leader) sm100::mbar_arrive_expect_tx(q_full, 2 * kQBytes);
          for (int c = 0; c < 4; ++c) pair_load_2d(&tm_q, qb, sQ + c * (BQ * 128), c * 64, m0 * kHeads, pol);
          ++nq;
        }
        if (ck.it < my_pairs &&
            (nk < kPairKSlots || sm100::mbar_test(sm100::smem_u32(&k_empty[k_s]), k_ph ^ 1))) {
          load_k();
          ++nk;
        }
        if (cv.it < my_pairs && nv < nk &&
            (nv < kPairVSlots || sm100::mbar_test(sm100::smem_u32(&v_empty[v_s]), v_ph ^ 1))) {
          load_v();
          ++nv;
        }
        if (clock64() - t0 > (1ll << 34)) {
          printf("sf: pair attention producer timeout (block %d)\n", blockIdx.x);
          __trap();
        }
      }
    }
  } else if (warp == 1) {
    if (leader && sm100::elect_one()) {
      const uint32_t idesc_s = sm100::make_idesc_bf16(256, 2 * BKEY);
      const uint32_t idesc_o = sm100::make_idesc_bf16(256, HD);
      const uint32_t q_addr = sm100::smem_u32(sQ);
      // One global superblock stream across pair tiles: S(g) then PV(g-1), so
      // the first S of the next tile is issued before the previous tile's
      // last PV and its softmax overlaps that PV; PV of a tile's first
      // superblock waits until the softmax warps drained the previous O.
      long long g = 0;  // global superblock counter
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;
      int pv_it = 0, pv_i = 0, pv_nsb = 0;  // tile / index of the next PV
      auto tile_nsb = [&](int t) {
        int env, env_start, m0, sb, nbt;
        bool valid;
        pair_geom(cl + t * n_cl, env, env_start, m0, valid, sb, nbt);
        return (nbt + 1) / 2;
      };
      auto issue_pv = [&](long long gg) {
        if (pv_i == 0 && pv_it > 0) sm100::mbar_wait(o_free, (pv_it - 1) & 1);
        sm100::mbar_wait(&p_full[gg & 1], (gg >> 1) & 1);
        sm100::mbar_wait(&v_full[vs], vph);
        sm100::tc_fence_after();
        const uint32_t v_addr = sm100::smem_u32(sV + vs * kPairVBytes);
        const uint32_t p_tmem = tmem + (uint32_t)(gg & 1) * (2 * BKEY);
#pragma unroll
        for (int kk = 0; kk < 2 * BKEY / 16; ++kk)  // 16 keys per MMA: 8 P columns, V^T chunk kk / 4
          pair_mma_ts(tmem + kPairOCol, p_tmem + kk * 8,
                      sm100::make_sw128_desc(v_addr + (kk >> 2) * (kPairVBytes / 2) + (kk & 3) * 32), idesc_o,
                      (pv_i | kk) != 0);
        pair_commit(&pv_done[gg & 1]);
        pair_commit(&v_empty[vs]);
        if (++vs == kPairVSlots) {
          vs = 0;
          vph ^= 1;
        }
        if (++pv_i == pv_nsb) {
          pv_i = 0;
          ++pv_it;
          if (pv_it < my_pairs) pv_nsb = tile_nsb(pv_it);
        }
      };
      if (my_pairs > 0) pv_nsb = tile_nsb(0);
      for (int it = 0; it < my_pairs; ++it) {
        const int nsb = tile_nsb(it);
        sm100::mbar_wait(q_full, it & 1);
        for (int i = 0; i < nsb; ++i, ++g) {
          sm100::mbar_wait(&k_full[ks], kph);
          sm100::tc_fence_after();
          const uint32_t k_addr = sm100::smem_u32(sK + ks * kPairKBytes);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const int c = kk >> 2, w = kk & 3;
            pair_mma(tmem + (uint32_t)(g & 1) * (2 * BKEY), sm100::make_sw128_desc(q_addr + c * (BQ * 128) + w * 32),
                     sm100::make_sw128_desc(k_addr + c * (BKEY * 128) + w * 32), idesc_s, kk != 0);
          }
          pair_commit(&s_full[g & 1]);
          pair_commit(&k_empty[ks]);
          if (++ks == kPairKSlots) {
            ks = 0;
            kph ^= 1;
          }
          if (i == nsb - 1) pair_commit(q_empty);
          if (g >= 1) issue_pv(g - 1);
        }
      }
      if (g > 0) issue_pv(g - 1);
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;  // keys [64 half, 64 half + 64) of a superblock = block 2G + half
    const int r = q * 32 + lane;
    const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t pfull_l = pair_mapa(sm100::smem_u32(p_full), 0);
    const uint32_t ofree_l = pair_mapa(sm100::smem_u32(o_free), 0);
    sm100::pdl_wait();
    if (threadIdx.x == 64) sm100::pdl_launch_dependents();
    long long g = 0;
    // A tile's O is drained after the NEXT tile's first superblock (whose S
    // the MMA issues before this tile's last PV), so that PV overlaps softmax.
    // xm slot for the row-sum exchange: glast & 1 when deferred (softmax of
    // glast + 1 synchronised in between), else the other slot.
    auto epilogue = [&](float lsum, int etok, bool estore, long long glast, bool deferred) {
      sm100::mbar_wait(&pv_done[glast & 1], (glast >> 1) & 1);
      sm100::tc_fence_after();
      const int ls = (int)((deferred ? glast : glast + 1) & 1);
      xm[(ls * 2 + half) * BQ + r] = lsum;
      asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
      lsum = xm[(ls * 2) * BQ + r] + xm[(ls * 2 + 1) * BQ + r];
      asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
      uint32_t ow[4][2][8];
#pragma unroll
      for (int u4 = 0; u4 < 4; ++u4) {
        uint32_t o[2][16];
        const int c0 = half * 128 + u4 * 32;
        sm100::tmem_ld16(t_lane + kPairOCol + c0, o[0]);
        sm100::tmem_ld16(t_lane + kPairOCol + c0 + 16, o[1]);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int kq = 0; kq < 8; ++kq) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(o[u][2 * kq]) * inv,
                                                      __uint_as_float(o[u][2 * kq + 1]) * inv);
            ow[u4][u][kq] = *reinterpret_cast<uint32_t*>(&b2);
          }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) pair_arrive(ofree_l);
      if (estore) {
        __nv_bfloat16* dst = p.out + (size_t)etok * (kHeads * HD) + (r & 7) * HD + half * 128;
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4)
#pragma unroll
          for (int u = 0; u < 2; ++u)  // 16 dims = one full 32 B sector per store
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + u4 * 32 + 16 * u),
                         "r"(ow[u4][u][0]), "r"(ow[u4][u][1]), "r"(ow[u4][u][2]), "r"(ow[u4][u][3]),
                         "r"(ow[u4][u][4]), "r"(ow[u4][u][5]), "r"(ow[u4][u][6]), "r"(ow[u4][u][7])
                         : "memory");
      }
    };
    bool pend = false, pend_store = false;
    float pend_lsum = 0.f;
    int pend_tok = 0;
    long long pend_glast = 0;
    for (int it = 0; it < my_pairs; ++it) {
      int env, env_start, m0, sb, nbt;
      bool valid;
      pair_geom(cl + it * n_cl, env, env_start, m0, valid, sb, nbt);
      const int nsb = (nbt + 1) / 2;
      const int tok = m0 + (r >> 3);
      const int head = r & 7;
      const int local_q = tok - env_start;
      const int seg_q = local_q / p.seg_len;
      const int t_q = local_q - seg_q * p.seg_len;
      const bool real_q = valid && local_q < p.segs * p.seg_len && tok < p.M;
      const bool store_q = valid && local_q < p.env_rows && tok < p.M;  // the row's token belongs to this env
      const int seg_lo = seg_q * p.seg_len;
      const int seg_hi = seg_lo + (t_q >= 1 ? p.seg_len : 1);
      float m_used = -INFINITY, l_sum = 0.f;
      for (int i = 0; i < nsb; ++i, ++g) {
        const int s = (int)(g & 1);
        const uint32_t t_s = t_lane + (uint32_t)s * (2 * BKEY);
        sm100::mbar_wait(&s_full[s], (g >> 1) & 1);
        sm100::tc_fence_after();
        float sv[64];
        {
          uint32_t raw[4][16];
#pragma unroll
          for (int c = 0; c < 4; ++c) sm100::tmem_ld16(t_s + half * BKEY + c * 16, raw[c]);
          sm100::tmem_ld_wait();
          const int j = 2 * i + half;
          int lo = 0, hi;
          if (j >= nbt) {
            hi = 0;
          } else if (j < p.n_prefix_blocks) {
            hi = p.prefix_len - j * BKEY;
          } else if (real_q) {
            const int base = sb + (j - p.n_prefix_blocks) * BKEY - env_start;
            lo = seg_lo - base;
            hi = seg_hi - base;
          } else {
            hi = 0;
          }
          if (lo <= 0 && hi >= BKEY) {
#pragma unroll
            for (int c = 0; c < 64; ++c) sv[c] = __uint_as_float(raw[c >> 4][c & 15]);
          } else {
#pragma unroll
            for (int c = 0; c < 64; ++c) {
              const float x = __uint_as_float(raw[c >> 4][c & 15]);
              sv[c] = (c >= lo && c < hi) ? x : -INFINITY;
            }
          }
        }
        float mb;
        {
          float t[22];
#pragma unroll
          for (int c = 0; c < 21; ++c) t[c] = fmax3(sv[3 * c], sv[3 * c + 1], sv[3 * c + 2]);
          t[21] = sv[63];
          float u[8];
#pragma unroll
          for (int c = 0; c < 7; ++c) u[c] = fmax3(t[3 * c], t[3 * c + 1], t[3 * c + 2]);
          u[7] = t[21];
          mb = fmaxf(fmax3(u[0], u[1], u[2]), fmaxf(fmax3(u[3], u[4], u[5]), fmaxf(u[6], u[7])));
        }
        // both halves of the row finished reading S (their tcgen05.ld waited)
        // before anyone overwrites the slot's first 64 columns with P
        xm[(s * 2 + half) * BQ + r] = mb;
        asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
        mb = fmaxf(xm[(s * 2) * BQ + r], xm[(s * 2 + 1) * BQ + r]) * p.scale_log2;
        const float m_new = fmaxf(m_used, mb);
        bool rescale = false;
        float alpha = 1.f;
        if (m_new > -INFINITY) {
          if (m_used == -INFINITY) {
            m_used = m_new;
          } else if (m_new > m_used + 8.f) {
            alpha = exp2f(m_used - m_new);
            m_used = m_new;
            rescale = true;
          }
        }
        const float mu = m_used == -INFINITY ? 0.f : m_used;
        uint32_t pw[32];
        float lp = 0.f;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float p0 = ex2_approx(fmaf(sv[2 * k], p.scale_log2, -mu));
          const float p1 = ex2_approx(fmaf(sv[2 * k + 1], p.scale_log2, -mu));
          lp += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          pw[k] = *reinterpret_cast<uint32_t*>(&b2);
        }
        const bool any_rescale = __any_sync(0xffffffffu, rescale);
        if (any_rescale && i >= 1) {
          sm100::mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
          sm100::tc_fence_after();
          l_sum *= alpha;
#pragma unroll 1
          for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 16) {
            uint32_t o[16];
            sm100::tmem_ld16(t_lane + kPairOCol + c0, o);
            sm100::tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
            sm100::tmem_st16(t_lane + kPairOCol + c0, o);
          }
          sm100::tmem_st_wait();
        } else if (rescale) {
          l_sum *= alpha;
        }
        l_sum += lp;
        // P(G) keys [64 half, +64) -> columns [32 half, 32 half + 32) of the slot
        sm100::tmem_st16(t_s + half * 32, *reinterpret_cast<const uint32_t(*)[16]>(&pw[0]));
        sm100::tmem_st16(t_s + half * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(&pw[16]));
        sm100::tmem_st_wait();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) pair_arrive(pfull_l + s * 8);
        if (i == 0 && pend) {
          epilogue(pend_lsum, pend_tok, pend_store, pend_glast, true);
          pend = false;
        }
      }
      pend = nsb > 0;
      pend_lsum = l_sum;
      pend_tok = tok;
      pend_store = store_q;
      pend_glast = g - 1;
    }
    if (pend) epilogue(pend_lsum, pend_tok, pend_store, pend_glast, false);
  }
  sm100::tc_fence_before();
  cluster.sync();  // the peer's barriers / TMEM are no longer referenced
  if (warp == 1) {
    sm100::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace attn
}  // namespace sf
