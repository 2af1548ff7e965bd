// Batch-1 layer-stack megakernel for the pi0-scale Action Expert (sm_100a).
//
// One persistent launch runs the whole Action Expert stack of a batch-1 round
// (<= 256 token rows): 18 x [QKV GEMM, MQA attention, O GEMM, gate/up GEMM,
// down GEMM] + the velocity head, as a sequence of PHASES separated by a
// grid-wide barrier (one CTA per SM, all co-resident). Each CTA runs at most
// one task per phase (task = blockIdx.x):
//   GEMM phase   swap-AB split-K tile (128 weight rows x all token rows x a
//                K range, tcgen05 with TMEM accumulator); the S split CTAs of
//                a tile exchange fp32 partials through L2 and meet on a
//                per-tile arrival counter, then each reduces 1/S of the
//                columns in a fixed split order (deterministic) and runs the
//                fused epilogue (RMS scale + RoPE, residual + RMS partials,
//                GeGLU, bias) -- the same epilogues as gemm.cuh.
//   ATTN phase   (16 tokens x 8 heads) query tile x a key-block range, QK^T
//                and PV on tcgen05 with online softmax (as attention.cuh);
//                split-KV partials merged through L2 after a per-tile counter.
// What the single launch buys over one kernel per op: no launch / ramp /
// drain per op, and the weights of phase p+1 stream into the SMEM ring (and
// the rest into L2) while phase p finishes its epilogue, reduction and the
// grid barrier -- weights never depend on activations.
//
// Barriers are initialised once and their phases tracked with running
// counters (k-blocks, key blocks, tasks), so no barrier is re-initialised
// while an asynchronous arrival may still be in flight. The data region
// (GEMM TMA ring | attention Q, K/V stages, P) is re-purposed per phase; the
// producer drains the previous phase's MMAs (empty barriers) before it
// issues loads for the next one.
#pragma once

#include "attention.cuh"
#include "gemm.cuh"

namespace sf {
namespace stack {

// 8 warps (2 per SM sub-partition, so up to 255 registers per thread): warp 0
// lane 0 issues TMA, warp 1 lane 0 issues tcgen05.mma; once the mainloop is
// issued every warp joins the epilogue (2 warps per TMEM lane quarter), and
// warps 4-7 run the attention softmax.
constexpr int kThreads = gemm::kEpiThreads;  // 256
constexpr uint32_t kRingMax = attn::kQBytes + 2 * attn::kStageBytes;    // 192 KB (P buffer after)
constexpr uint32_t kDataBytes = kRingMax + attn::kPBytes;               // 208 KB
constexpr int kMaxStages = 8;
constexpr int kMaxTileSlots = 64;  // per-phase split arrival counters

struct Ctl {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  uint64_t tmem_full;
  uint64_t q_full;
  uint64_t kv_full[2];
  uint64_t kv_empty[2];
  uint64_t s_full[2];
  uint64_t s_free[2];
  uint64_t p_full;
  uint64_t pv_done;
  uint32_t tmem_slot;
  uint32_t pad[3];
  float rs[256];
  float red[4 * 256];
  gemm::Params gp;           // current GEMM phase plan
  float xch[128 * 17];       // split-K: warp group 1 -> group 0 partial sums
  unsigned long long* dbg;   // trace context
  int n_phases, ph;
};
constexpr size_t kSmemBytes = 1024 + kDataBytes + ((sizeof(Ctl) + 127) & ~size_t(127));

enum PhaseKind : int { PH_GEMM = 0, PH_ATTN = 1 };
// GEMM phase types: the plan (geometry + fused epilogue) is the same for every
// layer, only the weight tensor map changes.
enum GemmType : int { T_QKV = 0, T_O = 1, T_GU = 2, T_DOWN = 3, T_HEAD = 4, T_COUNT = 5 };

// Everything lives in kernel-parameter space (constant bank): the per-type
// plans are read with compile-time indices inside the epilogues.
struct Args {
  gemm::Params gp[T_COUNT];        // per GEMM type (tiles_b == 1, splits, ws, epilogue)
  const CUtensorMap* tx[T_COUNT];  // activation map per type (B operand, bn-row box)
  const CUtensorMap* tw;           // weight maps [layers * 4 + 1] (qkv, o, gu, down per layer; head)
  const CUtensorMap* am;           // attention maps [layers][5] (q, k/v^T prefix, k/v^T suffix)
  int layers;
  int n_phases;             // 5 * layers + 1
  int attn_tasks;
  int stages;               // GEMM ring depth (fixed for the launch)
  uint32_t stage_bytes;     // A box + B box, 1 KB aligned
  uint32_t b_bytes;         // B box bytes (bn x 64 bf16)
  int bn;
  attn::Params ap;          // attention geometry (all layers)
  unsigned* grid_bar;       // [0] monotonic arrivals, [1] exits (re-armed by the last CTA)
  unsigned* tile_cnt;       // [n_phases][kMaxTileSlots] split arrivals
  unsigned long long* dbg;  // optional [grid][n_phases][8] %globaltimer stamps (null: off)
};

__device__ __forceinline__ void dstamp(const Args& a, int ph, int i) {
  if (a.dbg) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[((size_t)blockIdx.x * a.n_phases + ph) * 8 + i] = t;
  }
}

// Phase ph of the schedule: 5 per layer (QKV, ATTN, O, GU, DOWN), then HEAD.
struct PhaseRef {
  int kind, type, tasks;
  const CUtensorMap* tw;
  const CUtensorMap* tx;
  const CUtensorMap* am;
};

__device__ __forceinline__ PhaseRef phase_ref(const Args& a, int ph) {
  PhaseRef r;
  const int l = ph / 5, j = ph - 5 * (ph / 5);
  r.am = nullptr;
  r.tw = r.tx = nullptr;
  if (l >= a.layers) {
    r.kind = PH_GEMM;
    r.type = T_HEAD;
    r.tw = a.tw + 4 * a.layers;
  } else if (j == 1) {
    r.kind = PH_ATTN;
    r.type = -1;
    r.tasks = a.attn_tasks;
    r.am = a.am + 5 * l;
    return r;
  } else {
    r.kind = PH_GEMM;
    r.type = j == 0 ? T_QKV : j - 1;  // O = 1, GU = 2, DOWN = 3
    r.tw = a.tw + 4 * l + r.type;
  }
  r.tx = a.tx[r.type];
  r.tasks = a.gp[r.type].tiles_a * a.gp[r.type].splits;
  return r;
}

// ------------------------------------------------------------ sync helpers

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void spin_until(const unsigned* p, unsigned target, int what) {
  if (ld_acquire(p) >= target) return;
  const long long t0 = clock64();
  while (ld_acquire(p) < target) {
    __nanosleep(20);
    if (clock64() - t0 > (1ll << 33)) {
      printf("sf stack: %s barrier timeout (block %d, have %u want %u)\n",
             what ? "tile" : "grid", blockIdx.x, ld_acquire(p), target);
      __trap();
    }
  }
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// All threads: the CTA barrier orders every thread's stores of the phase
// before thread 0's release-add (cumulativity); the acquire-load on the other
// side orders them before the waiting CTA's reads (bar.sync again).
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_add(bar, 1u);
    spin_until(bar, target, 0);
  }
  __syncthreads();
}

// Epilogue warps (all 256 threads) of the S split CTAs of one tile meet here.
__device__ __forceinline__ void tile_sync(unsigned* cnt, unsigned target) {
  gemm::epi_bar();
  if (threadIdx.x == 64) {
    red_release_add(cnt, 1u);
    spin_until(cnt, target, 1);
  }
  gemm::epi_bar();
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* m, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 2, 128;" ::: "memory"); }

// ------------------------------------------------------------ GEMM pieces

__device__ __forceinline__ void cstamp(const Ctl& C, int i) {
  if (C.dbg) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    C.dbg[((size_t)blockIdx.x * C.n_phases + C.ph) * 8 + i] = t;
  }
}

struct GemmTask {
  int tile_a, split, kb0, nkb;
};

__device__ __forceinline__ GemmTask gemm_task(const gemm::Params& p, int task) {
  GemmTask t;
  t.tile_a = task % p.tiles_a;
  t.split = task / p.tiles_a;
  t.kb0 = t.split * p.kb_per_split;
  t.nkb = min(p.kb_per_split, p.num_kb - t.kb0);
  return t;
}

// Producer, before the grid barrier of the previous phase: weight tiles of
// the first ring slots (waiting for the previous MMAs to free them) + an L2
// prefetch of the rest. Returns the number of k-blocks pre-issued.
__device__ __forceinline__ int gemm_pre(const Args& a, const PhaseRef& P, uint8_t* data, Ctl& C,
                                        int kiter) {
  if ((int)blockIdx.x >= P.tasks) return 0;
  const GemmTask t = gemm_task(a.gp[P.type], blockIdx.x);
  const uint64_t pol_w = sm100::policy_evict_first();
  const int npre = min(a.stages, t.nkb);
  for (int i = 0; i < npre; ++i) {
    const int k = kiter + i;
    const int s = k % a.stages;
    if (k >= a.stages) sm100::mbar_wait(&C.empty[s], ((k / a.stages) & 1) ^ 1);
    sm100::mbar_arrive_expect_tx(&C.full[s], gemm::kAStageBytes + a.b_bytes);
    sm100::tma_load_2d(P.tw, &C.full[s], data + (size_t)s * a.stage_bytes, (t.kb0 + i) * gemm::BK,
                       t.tile_a * gemm::BM, pol_w);
  }
  for (int i = npre; i < t.nkb; ++i)
    tma_prefetch_l2(P.tw, (t.kb0 + i) * gemm::BK, t.tile_a * gemm::BM);
  return npre;
}

// Producer, after the grid barrier: activation tiles of the pre-issued
// slots, then whole stages for the rest of the K range.
__device__ __noinline__ void gemm_post(const Args& a, const PhaseRef& P, uint8_t* data, Ctl& C,
                                          int& kiter, int npre) {
  if ((int)blockIdx.x >= P.tasks) return;
  const GemmTask t = gemm_task(a.gp[P.type], blockIdx.x);
  const uint64_t pol_w = sm100::policy_evict_first();
  const uint64_t pol_x = sm100::policy_evict_last();
  fence_proxy_async_global();
  for (int i = 0; i < npre; ++i) {
    const int s = (kiter + i) % a.stages;
    sm100::tma_load_2d(P.tx, &C.full[s], data + (size_t)s * a.stage_bytes + gemm::kAStageBytes,
                       (t.kb0 + i) * gemm::BK, 0, pol_x);
  }
  for (int i = npre; i < t.nkb; ++i) {
    const int k = kiter + i;
    const int s = k % a.stages;
    if (k >= a.stages) sm100::mbar_wait(&C.empty[s], ((k / a.stages) & 1) ^ 1);
    uint8_t* st = data + (size_t)s * a.stage_bytes;
    sm100::mbar_arrive_expect_tx(&C.full[s], gemm::kAStageBytes + a.b_bytes);
    sm100::tma_load_2d(P.tw, &C.full[s], st, (t.kb0 + i) * gemm::BK, t.tile_a * gemm::BM, pol_w);
    sm100::tma_load_2d(P.tx, &C.full[s], st + gemm::kAStageBytes, (t.kb0 + i) * gemm::BK, 0, pol_x);
  }
  kiter += t.nkb;
}

// Producer: wait until every MMA that read the ring has retired (the data
// region is about to be re-purposed for attention).
__device__ __forceinline__ void gemm_drain(const Args& a, Ctl& C, int kiter) {
  for (int k = max(0, kiter - a.stages); k < kiter; ++k)
    sm100::mbar_wait(&C.empty[k % a.stages], (k / a.stages) & 1);
}

__device__ __noinline__ void gemm_mma(const Args& a, const PhaseRef& P, uint8_t* data, Ctl& C,
                                         uint32_t tmem, int& kiter) {
  if ((int)blockIdx.x >= P.tasks) return;
  const GemmTask t = gemm_task(a.gp[P.type], blockIdx.x);
  const uint32_t idesc = sm100::make_idesc_bf16(gemm::BM, a.bn);
  for (int i = 0; i < t.nkb; ++i) {
    const int k = kiter + i;
    const int s = k % a.stages;
    sm100::mbar_wait(&C.full[s], (k / a.stages) & 1);
    sm100::tc_fence_after();
    const uint32_t a_addr = sm100::smem_u32(data + (size_t)s * a.stage_bytes);
    const uint32_t b_addr = a_addr + gemm::kAStageBytes;
#pragma unroll
    for (int kk = 0; kk < gemm::BK / 16; ++kk)
      sm100::umma_bf16(tmem, sm100::make_sw128_desc(a_addr + kk * 32),
                       sm100::make_sw128_desc(b_addr + kk * 32), idesc, (i | kk) != 0);
    sm100::umma_commit(&C.empty[s]);
  }
  sm100::umma_commit(&C.tmem_full);
  kiter += t.nkb;
}

// Epilogue warps (2-9): row scales, accumulator -> (split-K partial, tile
// counter, reduction) -> fused epilogue. Same data layouts as gemm.cuh.
template <int KIND>
__device__ __forceinline__ void gemm_epilogue(const gemm::Params& p, Ctl& C, uint32_t tmem,
                                              int gtask, unsigned* tile_cnt) {
  const gemm::EpiArgs& e = p.e;
  const GemmTask t = gemm_task(p, blockIdx.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;
  const int g = warp >> 2;
  const int lane_row = q * 32 + lane;
  const int n = t.tile_a * gemm::BM + lane_row;
  const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
  for (int c = threadIdx.x; c < p.bn; c += gemm::kEpiThreads)
    C.rs[c] = (KIND != gemm::EPI_RESID && KIND != gemm::EPI_TANH_BF16 && c < e.M) ? gemm::row_scale(e, c) : 1.f;
  sm100::mbar_wait(&C.tmem_full, gtask & 1);
  sm100::tc_fence_after();
  if (threadIdx.x == 64) cstamp(C, 3);
  const int nchunks = p.bn / 16;
  const int S = p.splits;
  if (S == 1) {
    gemm::epi_bar();
    for (int ch = g; ch < nchunks; ch += 4) {
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
        gemm::epi_swap<KIND>(e, n, c * 16, v, C.rs, C.red + q * 256, c * 16);
      }
    }
    if (KIND == gemm::EPI_RESID) {
      gemm::epi_bar();
      for (int c = threadIdx.x; c < p.bn; c += gemm::kEpiThreads)
        if (c < e.M)
          e.ssq_out[(size_t)t.tile_a * e.ssq_out_ld + c] =
              ((C.red[c] + C.red[256 + c]) + C.red[512 + c]) + C.red[768 + c];
    }
    return;
  }
  const int tile_id = t.tile_a;  // tiles_b == 1
  const size_t slab = (size_t)nchunks * gemm::BM * 16;
  float* mine = p.ws + ((size_t)t.split * p.total_tiles + tile_id) * slab;
  for (int ch = g; ch < nchunks; ch += 8) {
    uint32_t r[4][16];
    // unconditional loads (columns past bn are allocated, just unused)
#pragma unroll
    for (int u = 0; u < 4; ++u) sm100::tmem_ld16(t_lane + (ch + 2 * u) * 16, r[u]);
    sm100::tmem_ld_wait();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (ch + 2 * u >= nchunks) break;
      float4* dst = reinterpret_cast<float4*>(mine + (size_t)(ch + 2 * u) * gemm::BM * 16) + lane_row;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        __stcg(dst + j * gemm::BM,
               make_float4(__uint_as_float(r[u][4 * j]), __uint_as_float(r[u][4 * j + 1]),
                           __uint_as_float(r[u][4 * j + 2]), __uint_as_float(r[u][4 * j + 3])));
    }
  }
  if (threadIdx.x == 64) cstamp(C, 7);
  tile_sync(tile_cnt + tile_id, (unsigned)S);
  if (threadIdx.x == 64) cstamp(C, 4);
  const float* base = p.ws + (size_t)tile_id * slab + lane_row * 4;
  const size_t sstride = (size_t)p.total_tiles * slab;
  // Owned chunks ch = split + k * S. Both warp groups work on the same chunk:
  // group 0 sums splits [0, S/2), group 1 splits [S/2, S), every load of a
  // group in flight at once; group 1 hands its sum over SMEM, group 0 adds it
  // (fixed order: deterministic) and runs the fused epilogue.
  float* xch = C.xch + lane_row * 17;
  const int half = (S + 1) >> 1;
  const int s_lo = g ? half : 0, s_hi = g ? S : half;
  for (int ch = t.split; ch < nchunks; ch += S) {
    const float4* ps = reinterpret_cast<const float4*>(base + (size_t)ch * gemm::BM * 16);
    float4 acc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = s_lo; s0 < s_hi; s0 += 8) {
      float4 v[8][4];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int su = min(s0 + u, s_hi - 1);  // unconditional loads keep v in registers
#pragma unroll
        for (int j = 0; j < 4; ++j) v[u][j] = __ldcg(ps + (size_t)su * (sstride / 4) + j * gemm::BM);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < s_hi)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[j].x += v[u][j].x;
            acc[j].y += v[u][j].y;
            acc[j].z += v[u][j].z;
            acc[j].w += v[u][j].w;
          }
    }
    if (g == 1) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        xch[4 * j] = acc[j].x;
        xch[4 * j + 1] = acc[j].y;
        xch[4 * j + 2] = acc[j].z;
        xch[4 * j + 3] = acc[j].w;
      }
    }
    gemm::epi_bar();
    if (g == 0) {
      float vv[16];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        vv[4 * j] = acc[j].x + xch[4 * j];
        vv[4 * j + 1] = acc[j].y + xch[4 * j + 1];
        vv[4 * j + 2] = acc[j].z + xch[4 * j + 2];
        vv[4 * j + 3] = acc[j].w + xch[4 * j + 3];
      }
      gemm::epi_swap<KIND>(e, n, ch * 16, vv, C.rs, C.red + q * 256, ch * 16);
    }
    gemm::epi_bar();
  }
  if (KIND == gemm::EPI_RESID) {
    gemm::epi_bar();
    for (int c = threadIdx.x; c < p.bn; c += gemm::kEpiThreads)
      if ((c >> 4) % S == t.split && c < e.M)
        e.ssq_out[(size_t)t.tile_a * e.ssq_out_ld + c] =
            ((C.red[c] + C.red[256 + c]) + C.red[512 + c]) + C.red[768 + c];
  }
}

__device__ __forceinline__ void gemm_epilogue_any(const Args& a, const PhaseRef& P, Ctl& C,
                                                  uint32_t tmem, int gtask, unsigned* tile_cnt) {
  switch (P.type) {
    case T_QKV: gemm_epilogue<gemm::EPI_QKV>(C.gp, C, tmem, gtask, tile_cnt); break;
    case T_O:
    case T_DOWN: gemm_epilogue<gemm::EPI_RESID>(C.gp, C, tmem, gtask, tile_cnt); break;
    case T_GU: gemm_epilogue<gemm::EPI_GEGLU>(C.gp, C, tmem, gtask, tile_cnt); break;
    case T_HEAD: gemm_epilogue<gemm::EPI_F32>(C.gp, C, tmem, gtask, tile_cnt); break;
    default: break;
  }
}

// ------------------------------------------------------------ attention pieces

struct AttnTask {
  int tile, split, m0, env_start, sb, j0, nb;
};

__device__ __forceinline__ AttnTask attn_task(const attn::Params& p, int task) {
  AttnTask t;
  t.tile = task % p.tiles;
  t.split = task / p.tiles;
  t.m0 = t.tile * 16;
  const int env = t.m0 / p.env_rows;
  t.env_start = env * p.env_rows;
  const int seg_first = (t.m0 - t.env_start) / p.seg_len;
  t.sb = (t.env_start + seg_first * p.seg_len) & ~(attn::BKEY - 1);
  t.j0 = t.split * p.blocks_per_split;
  t.nb = max(0, min(p.blocks_per_split, p.n_blocks - t.j0));
  return t;
}

struct AttnSmem {
  uint8_t* q;
  uint8_t* kv;
  uint8_t* pbuf;
};

__device__ __forceinline__ AttnSmem attn_smem(uint8_t* data) {
  return AttnSmem{data, data + attn::kQBytes, data + attn::kQBytes + 2 * attn::kStageBytes};
}

// Issue key block i (global block counter g) of task t; false when the block
// is a suffix block and only prefix blocks are allowed (before the barrier).
__device__ __forceinline__ bool attn_load_block(const Args& a, const PhaseRef& P, const AttnTask& t,
                                                const AttnSmem& sm, Ctl& C, int i, int g,
                                                bool prefix_only) {
  const int j = t.j0 + i;
  const bool is_prefix = j < a.ap.n_prefix_blocks;
  if (prefix_only && !is_prefix) return false;
  const int s = g & 1;
  if (g >= 2) sm100::mbar_wait(&C.kv_empty[s], ((g >> 1) & 1) ^ 1);
  uint8_t* st = sm.kv + s * attn::kStageBytes;
  const uint64_t pol = sm100::policy_evict_last();
  sm100::mbar_arrive_expect_tx(&C.kv_full[s], attn::kStageBytes);
  const int env = a.ap.env_map ? __ldg(a.ap.env_map + t.env_start / a.ap.env_rows)
                                : t.env_start / a.ap.env_rows;
  if (is_prefix) {
    for (int c = 0; c < 4; ++c)
      attn::tma_load_3d(&P.am[1], &C.kv_full[s], st + c * (attn::BKEY * 128), c * 64, j * attn::BKEY,
                        env, pol);
    attn::tma_load_3d(&P.am[2], &C.kv_full[s], st + attn::kKBytes, j * attn::BKEY, 0, env, pol);
  } else {
    const int row0 = t.sb + (j - a.ap.n_prefix_blocks) * attn::BKEY;
    for (int c = 0; c < 4; ++c)
      sm100::tma_load_2d(&P.am[3], &C.kv_full[s], st + c * (attn::BKEY * 128), c * 64, row0, pol);
    sm100::tma_load_2d(&P.am[4], &C.kv_full[s], st + attn::kKBytes, row0, 0, pol);
  }
  return true;
}

__device__ __forceinline__ int attn_pre(const Args& a, const PhaseRef& P, uint8_t* data, Ctl& C,
                                        int akb) {
  if ((int)blockIdx.x >= P.tasks) return 0;
  const AttnTask t = attn_task(a.ap, blockIdx.x);
  const AttnSmem sm = attn_smem(data);
  int issued = 0;
  while (issued < min(2, t.nb) && attn_load_block(a, P, t, sm, C, issued, akb + issued, true)) ++issued;
  return issued;
}

__device__ __noinline__ void attn_post(const Args& a, const PhaseRef& P, uint8_t* data, Ctl& C,
                                          int& akb, int npre) {
  if ((int)blockIdx.x >= P.tasks) return;
  const AttnTask t = attn_task(a.ap, blockIdx.x);
  const AttnSmem sm = attn_smem(data);
  fence_proxy_async_global();
  const uint64_t pol = sm100::policy_evict_last();
  sm100::mbar_arrive_expect_tx(&C.q_full, attn::kQBytes);
  for (int c = 0; c < 4; ++c)
    sm100::tma_load_2d(&P.am[0], &C.q_full, sm.q + c * (attn::BQ * 128), c * 64, t.m0 * attn::kHeads,
                       pol);
  for (int i = npre; i < t.nb; ++i) attn_load_block(a, P, t, sm, C, i, akb + i, false);
  // drain: the data region is re-purposed by the next phase
  for (int i = max(0, t.nb - 2); i < t.nb; ++i) {
    const int g = akb + i;
    sm100::mbar_wait(&C.kv_empty[g & 1], (g >> 1) & 1);
  }
  akb += t.nb;
}

__device__ __noinline__ void attn_mma(const Args& a, const PhaseRef& P, uint8_t* data, Ctl& C,
                                         uint32_t tmem, int& akb, int atask) {
  if ((int)blockIdx.x >= P.tasks) return;
  const AttnTask t = attn_task(a.ap, blockIdx.x);
  const AttnSmem sm = attn_smem(data);
  const uint32_t idesc_s = sm100::make_idesc_bf16(attn::BQ, attn::BKEY);
  const uint32_t idesc_o = sm100::make_idesc_bf16(attn::BQ, attn::HD);
  const uint32_t q_addr = sm100::smem_u32(sm.q);
  const uint32_t p_addr = sm100::smem_u32(sm.pbuf);
  sm100::mbar_wait(&C.q_full, atask & 1);
  auto issue_pv = [&](int i) {
    const int g = akb + i;
    sm100::mbar_wait(&C.p_full, g & 1);
    sm100::tc_fence_after();
    const uint32_t v_addr = sm100::smem_u32(sm.kv + (g & 1) * attn::kStageBytes + attn::kKBytes);
#pragma unroll
    for (int kk = 0; kk < attn::BKEY / 16; ++kk)
      sm100::umma_bf16(tmem + 128, sm100::make_sw128_desc(p_addr + kk * 32),
                       sm100::make_sw128_desc(v_addr + kk * 32), idesc_o, (i | kk) != 0);
    sm100::umma_commit(&C.pv_done);
    sm100::umma_commit(&C.kv_empty[g & 1]);
  };
  for (int i = 0; i < t.nb; ++i) {
    const int g = akb + i;
    const int s = g & 1;
    sm100::mbar_wait(&C.kv_full[s], (g >> 1) & 1);
    if (g >= 2) sm100::mbar_wait(&C.s_free[s], ((g >> 1) & 1) ^ 1);
    sm100::tc_fence_after();
    const uint32_t k_addr = sm100::smem_u32(sm.kv + s * attn::kStageBytes);
#pragma unroll
    for (int kk = 0; kk < attn::HD / 16; ++kk) {
      const int c = kk >> 2, w = kk & 3;
      sm100::umma_bf16(tmem + s * attn::BKEY,
                       sm100::make_sw128_desc(q_addr + c * (attn::BQ * 128) + w * 32),
                       sm100::make_sw128_desc(k_addr + c * (attn::BKEY * 128) + w * 32), idesc_s,
                       kk != 0);
    }
    sm100::umma_commit(&C.s_full[s]);
    if (i >= 1) issue_pv(i - 1);
  }
  if (t.nb > 0) issue_pv(t.nb - 1);
  akb += t.nb;
}

// Softmax warps (2-5): online softmax over the task's key blocks; returns the
// row's final (m, l); O stays in TMEM columns [128, 384).
__device__ __forceinline__ void attn_softmax(const Args& a, const AttnTask& t, uint8_t* data, Ctl& C,
                                             uint32_t tmem, int akb, float& m_fin, float& l_fin) {
  const attn::Params& p = a.ap;
  const AttnSmem sm = attn_smem(data);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;
  const int r = q * 32 + lane;
  const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
  const int tok = t.m0 + (r >> 3);
  const int local_q = tok - t.env_start;
  const int seg_q = local_q / p.seg_len;
  const int t_q = local_q - seg_q * p.seg_len;
  const bool real_q = local_q < p.segs * p.seg_len && tok < p.M;
  const int seg_lo = seg_q * p.seg_len;
  const int seg_hi = seg_lo + (t_q >= 1 ? p.seg_len : 1);
  float m_used = -INFINITY, l_sum = 0.f;
  for (int i = 0; i < t.nb; ++i) {
    const int j = t.j0 + i;
    const int g = akb + i;
    const int s = g & 1;
    sm100::mbar_wait(&C.s_full[s], (g >> 1) & 1);
    sm100::tc_fence_after();
    uint32_t raw[4][16];
#pragma unroll
    for (int c = 0; c < 4; ++c) sm100::tmem_ld16(t_lane + s * attn::BKEY + c * 16, raw[c]);
    sm100::tmem_ld_wait();
    sm100::tc_fence_before();
    sm100::mbar_arrive(&C.s_free[s]);
    int lo = 0, hi;
    if (j < p.n_prefix_blocks) {
      hi = p.prefix_len - j * attn::BKEY;
    } else if (real_q) {
      const int base = t.sb + (j - p.n_prefix_blocks) * attn::BKEY - t.env_start;
      lo = seg_lo - base;
      hi = seg_hi - base;
    } else {
      hi = 0;
    }
    float sv[64];
    float mb = -INFINITY;
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      const float x = __uint_as_float(raw[c >> 4][c & 15]) * p.scale_log2;
      sv[c] = (c >= lo && c < hi) ? x : -INFINITY;
      mb = fmaxf(mb, sv[c]);
    }
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
    if (i >= 1) {
      sm100::mbar_wait(&C.pv_done, (g - 1) & 1);
      sm100::tc_fence_after();
    }
    if (__any_sync(0xffffffffu, rescale) && i >= 1) {
      l_sum *= alpha;
#pragma unroll 1
      for (int c0 = 0; c0 < attn::HD; c0 += 16) {
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
    uint8_t* prow = sm.pbuf + r * 128;
    const float mu = m_used == -INFINITY ? 0.f : m_used;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float p0 = exp2f(sv[c * 8 + 2 * k] - mu);
        const float p1 = exp2f(sv[c * 8 + 2 * k + 1] - mu);
        l_sum += p0 + p1;
        __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
        w[k] = *reinterpret_cast<uint32_t*>(&b2);
      }
      *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    attn::fence_async_smem();
    sm100::tc_fence_before();
    sm100::mbar_arrive(&C.p_full);
  }
  if (t.nb > 0) {
    sm100::mbar_wait(&C.pv_done, (akb + t.nb - 1) & 1);
    sm100::tc_fence_after();
  }
  m_fin = m_used;
  l_fin = l_sum;
}

// Epilogue warps (2-9) of an attention task: final output (1 split) or
// partial -> tile counter -> merge (as attention.cuh's L2 merge).
__device__ __forceinline__ void attn_epilogue(const Args& a, const AttnTask& t, uint8_t* data,
                                              Ctl& C, uint32_t tmem, float m_fin, float l_fin,
                                              unsigned* tile_cnt) {
  const attn::Params& p = a.ap;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool softmax_warp = warp >= 4;
  const int q = warp & 3;
  const int r = q * 32 + lane;
  const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
  const int S = p.splits;
  using attn::BQ;
  using attn::HD;
  if (S == 1) {
    if (!softmax_warp) return;
    const int tok = t.m0 + (r >> 3), head = r & 7;
    const float inv = l_fin > 0.f ? 1.f / l_fin : 0.f;
    __nv_bfloat16* dst = p.out + (size_t)tok * (attn::kHeads * HD) + head * HD;
    for (int c0 = 0; c0 < HD; c0 += 16) {
      uint32_t o[16];
      sm100::tmem_ld16(t_lane + 128 + c0, o);
      sm100::tmem_ld_wait();
      uint32_t w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) w[k] = gemm::pack_bf16(__uint_as_float(o[2 * k]) * inv, __uint_as_float(o[2 * k + 1]) * inv);
      if (tok < p.M) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
        d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
        d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
    return;
  }
  const int rows = (BQ + S - 1) / S;
  const int my_r0 = t.split * rows;
  const int my_nr = max(0, min(BQ, my_r0 + rows) - my_r0);
  const size_t part_floats = (size_t)HD * BQ;
  float4* ws_o = reinterpret_cast<float4*>(p.ws);
  float2* ws_ml = reinterpret_cast<float2*>(p.ws + (size_t)p.tiles * S * part_floats);
  if (softmax_warp) {
    float4* dst = ws_o + (size_t)(t.tile * S + t.split) * (HD / 4) * BQ + r;
    ws_ml[(size_t)(t.tile * S + t.split) * BQ + r] = make_float2(m_fin, l_fin);
#pragma unroll 1
    for (int c0 = 0; c0 < HD; c0 += 64) {
      uint32_t o[4][16];
#pragma unroll
      for (int u = 0; u < 4; ++u) sm100::tmem_ld16(t_lane + 128 + c0 + 16 * u, o[u]);
      sm100::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < 16; k += 4)
          __stcg(dst + (size_t)((c0 + 16 * u + k) >> 2) * BQ,
                 make_float4(__uint_as_float(o[u][k]), __uint_as_float(o[u][k + 1]),
                             __uint_as_float(o[u][k + 2]), __uint_as_float(o[u][k + 3])));
    }
  }
  if (threadIdx.x == 64) cstamp(C, 7);
  tile_sync(tile_cnt + t.tile, (unsigned)S);
  if (threadIdx.x == 64) cstamp(C, 4);
  const AttnSmem sm = attn_smem(data);
  // merge scratch in the P buffer (16 KB): rows <= 64 when S >= 2
  float* wgt = reinterpret_cast<float*>(sm.pbuf);  // [64][kMaxSplitsKV]
  float* inv = wgt + 64 * attn::kMaxSplitsKV;      // [64]
  const int et = threadIdx.x;  // 0..255
  if (et < my_nr) {
    const int row = my_r0 + et;
    float* lsv = inv + 64;  // [64][kMaxSplitsKV] l of each split
    float mx = -INFINITY;
    for (int s2 = 0; s2 < S; ++s2) {
      const float2 ml = __ldcg(ws_ml + (size_t)(t.tile * S + s2) * BQ + row);
      wgt[et * attn::kMaxSplitsKV + s2] = ml.x;
      lsv[et * attn::kMaxSplitsKV + s2] = ml.y;
      mx = fmaxf(mx, ml.x);
    }
    float L = 0.f;
    for (int s2 = 0; s2 < S; ++s2) {
      const float ms = wgt[et * attn::kMaxSplitsKV + s2];
      const float w = ms > -INFINITY ? exp2f(ms - mx) : 0.f;
      wgt[et * attn::kMaxSplitsKV + s2] = w;
      L += w * lsv[et * attn::kMaxSplitsKV + s2];
    }
    inv[et] = L > 0.f ? 1.f / L : 0.f;
  }
  gemm::epi_bar();
  const int total = my_nr * (HD / 4);
  constexpr int SG = 8;  // split loads in flight per output (x2 outputs)
  for (int idx0 = et; idx0 < total; idx0 += 2 * gemm::kEpiThreads) {
    float4 acc[2];
    acc[0] = acc[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < S; s0 += SG) {
      float4 v[2][SG];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int idx = idx0 + u * gemm::kEpiThreads;
        if (idx < total) {
          const int rr = idx % my_nr, c4 = idx / my_nr;
#pragma unroll
          for (int s2 = 0; s2 < SG; ++s2)
            if (s0 + s2 < S)
              v[u][s2] = __ldcg(ws_o + ((size_t)(t.tile * S + s0 + s2) * (HD / 4) + c4) * BQ + my_r0 + rr);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int idx = idx0 + u * gemm::kEpiThreads;
        if (idx < total) {
          const int rr = idx % my_nr;
#pragma unroll
          for (int s2 = 0; s2 < SG; ++s2)
            if (s0 + s2 < S) {
              const float w = wgt[rr * attn::kMaxSplitsKV + s0 + s2];
              acc[u].x += w * v[u][s2].x;
              acc[u].y += w * v[u][s2].y;
              acc[u].z += w * v[u][s2].z;
              acc[u].w += w * v[u][s2].w;
            }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int idx = idx0 + u * gemm::kEpiThreads;
      if (idx < total) {
        const int rr = idx % my_nr, c4 = idx / my_nr;
        const float iv = inv[rr];
        const int row = my_r0 + rr;
        const int tok = t.m0 + (row >> 3), head = row & 7;
        if (tok < p.M) {
          uint2 pk = make_uint2(gemm::pack_bf16(acc[u].x * iv, acc[u].y * iv),
                                gemm::pack_bf16(acc[u].z * iv, acc[u].w * iv));
          *reinterpret_cast<uint2*>(p.out + (size_t)tok * (attn::kHeads * HD) + head * HD + 4 * c4) = pk;
        }
      }
    }
  }
}

// ------------------------------------------------------------ the kernel

__device__ __noinline__ int phase_pre(const Args& a, int ph, uint8_t* data, Ctl& C, int kiter,
                                         int akb, int prev_kind) {
  const PhaseRef P = phase_ref(a, ph);
  if (P.kind == PH_GEMM) return gemm_pre(a, P, data, C, kiter);
  if (prev_kind == PH_GEMM) gemm_drain(a, C, kiter);
  return attn_pre(a, P, data, C, akb);
}

__global__ void __launch_bounds__(kThreads, 1) stack_kernel(const __grid_constant__ Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* data = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  Ctl& C = *reinterpret_cast<Ctl*>(data + kDataBytes);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      sm100::mbar_init(&C.full[s], 1);
      sm100::mbar_init(&C.empty[s], 1);
    }
    sm100::mbar_init(&C.tmem_full, 1);
    sm100::mbar_init(&C.q_full, 1);
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&C.kv_full[s], 1);
      sm100::mbar_init(&C.kv_empty[s], 1);
      sm100::mbar_init(&C.s_full[s], 1);
      sm100::mbar_init(&C.s_free[s], 128);
    }
    sm100::mbar_init(&C.p_full, 128);
    sm100::mbar_init(&C.pv_done, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<512>(&C.tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = C.tmem_slot;

  // running counters (every role advances its own copy along the same schedule)
  int kiter = 0, gtask = 0, akb = 0, atask = 0, npre = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4 * a.layers + 1; ++i) sm100::tma_prefetch_desc(a.tw + i);
    for (int i = 0; i < T_COUNT; ++i) sm100::tma_prefetch_desc(a.tx[i]);
    npre = phase_pre(a, 0, data, C, kiter, akb, -1);
  }
  sm100::pdl_wait();  // embed output (X, ssq) of the previous kernel

  for (int ph = 0; ph < a.n_phases; ++ph) {
    const PhaseRef P = phase_ref(a, ph);
    const bool active = (int)blockIdx.x < P.tasks;
    // this phase's GEMM plan -> SMEM: the epilogue reads its fields on demand
    // (held in registers across the phase loop they would spill)
    if (P.kind == PH_GEMM) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(&a.gp[P.type]);
      uint32_t* dst = reinterpret_cast<uint32_t*>(&C.gp);
      for (int i = threadIdx.x; i < (int)(sizeof(gemm::Params) / 4); i += kThreads) dst[i] = src[i];
    }
    if (threadIdx.x == 0) {
      C.dbg = a.dbg;
      C.n_phases = a.n_phases;
      C.ph = ph;
    }
    __syncthreads();
    unsigned* tcnt = a.tile_cnt + (size_t)ph * kMaxTileSlots;
    if (threadIdx.x == 0) dstamp(a, ph, 0);
    if (P.kind == PH_GEMM) {
      if (threadIdx.x == 0) {
        gemm_post(a, P, data, C, kiter, npre);
        dstamp(a, ph, 1);
        if (ph + 1 < a.n_phases) npre = phase_pre(a, ph + 1, data, C, kiter, akb, PH_GEMM);
      } else if (threadIdx.x == 32) {
        gemm_mma(a, P, data, C, tmem, kiter);
        dstamp(a, ph, 2);
      }
      __syncwarp();
      if (active) {
        gemm_epilogue_any(a, P, C, tmem, gtask, tcnt);
        if (threadIdx.x == 64) dstamp(a, ph, 5);
        ++gtask;
      }
    } else {
      if (threadIdx.x == 0) {
        attn_post(a, P, data, C, akb, npre);
        dstamp(a, ph, 1);
        if (ph + 1 < a.n_phases) npre = phase_pre(a, ph + 1, data, C, kiter, akb, PH_ATTN);
      } else if (threadIdx.x == 32) {
        attn_mma(a, P, data, C, tmem, akb, atask);
        dstamp(a, ph, 2);
      }
      __syncwarp();
      if (active) {
        const AttnTask t = attn_task(a.ap, blockIdx.x);
        float m_fin = -INFINITY, l_fin = 0.f;
        if (warp >= 4) {
          attn_softmax(a, t, data, C, tmem, akb, m_fin, l_fin);
          akb += t.nb;
          if (threadIdx.x == 128) dstamp(a, ph, 3);
        }
        attn_epilogue(a, t, data, C, tmem, m_fin, l_fin, tcnt);
        if (threadIdx.x == 64) dstamp(a, ph, 5);
        ++atask;
      }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) dstamp(a, ph, 6);
    grid_sync(a.grid_bar, (unsigned)(ph + 1) * gridDim.x);
    sm100::tc_fence_after();
  }
  if (threadIdx.x == 0) sm100::pdl_launch_dependents();
  // the last CTA out re-arms the counters for the next launch (every CTA has
  // left the final grid barrier once it bumped `exit`)
  __shared__ unsigned last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.grid_bar + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    for (int i = threadIdx.x; i < a.n_phases * kMaxTileSlots; i += blockDim.x) a.tile_cnt[i] = 0u;
    if (threadIdx.x == 0) {
      a.grid_bar[0] = 0u;
      a.grid_bar[1] = 0u;
    }
  }
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem);
  }
}

}  // namespace stack
}  // namespace sf
