// Batch-1 Euler full path as ONE persistent launch (sm_100a).
//
// flowpolicy.integrate_flow (flowpolicy.py:273-292) for one env at pi0 scale:
// N x [embed, 18 x (QKV, attention, O, gate/up, down), head] + the Euler
// update, as a sequence of STAGES separated by a grid barrier
// (one CTA per SM, cooperative launch). Why one launch: at batch 1 every
// layer op is a few MB of weights against 51 token rows, so the per-op
// kernels of the graph path are latency-bound (~9 us each: launch, ramp,
// split-K partials through L2, cluster barrier, reduction, epilogue). Here
//   * the weights never depend on activations: warp 0 of every CTA streams
//     its share of the NEXT stages' weights (and the prefix K/V block images
//     of its attention tasks) into a 4 x 32 KB TMA ring while the current
//     stage, the barrier and the activation loads run;
//   * split-K partials are reduced IN L2 with red.global.add.v4.f32 into fp32
//     accumulators (X, QKV, gate/up, head) -- no partial buffers, no tile
//     counters, no second pass (measured: 39 GB/s per SM, 1.2 us barrier,
//     profiles/r2/b1_primitives_microbench.log);
//   * the split CTAs of an output tile meet on a per-tile arrival counter;
//     the LAST one runs the tile's epilogue from the finished L2 sums (RMS
//     scale + RoPE -> bf16 q/k/v^T; GeGLU -> bf16 h; residual -> bf16 x +
//     RMS partial sums), so every GEMM operand of the next stage is a bf16
//     TMA load; the split-KV attention partials are merged by the O GEMM's
//     operand loader (the only worker-built operand).
// Rounding points are the device path's (oracle/pi0_oracle.py precision
// model): bf16 GEMM operands, fp32 accumulation and residual, bf16 q/k/v, P,
// o, h; the split-KV partial o is additionally stored as bf16 (normalised).
// The fp32 summation order of split-K differs run to run (L2 atomics).
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA
// issuer (one elected lane), warps 2-9 = 256 workers (operand transforms,
// accumulator epilogues with v4 L2 reductions, attention softmax: two warps
// per TMEM lane quarter, 32 of a key block's 64 columns each).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "sm100.cuh"

namespace sf {
namespace b1 {

using bf16 = __nv_bfloat16;

constexpr int kMaxL = 32;
constexpr int kGrid = 148;     // one CTA per SM (B200)
constexpr int kThreads = 320;
constexpr int kWorkers = 256;
constexpr int kTok = 64;       // UMMA N: token rows (T <= 64 real)
constexpr int kSlots = 4;
constexpr uint32_t kSlotBytes = 32768;  // one ring item: 2 k-blocks of 128 weight rows, or a K / V^T key block
constexpr uint32_t kRingBytes = kSlots * kSlotBytes;
constexpr uint32_t kBBytes = 65536;     // GEMM B operand (<= 8 k-blocks of 64 tokens) | attention Q | epilogue staging
constexpr uint32_t kCtlBytes = 8192 + 16384;  // barriers + scratch | the QKV tile's RoPE slice (16 KB)
constexpr uint32_t kSmemBytes = 1024 + kRingBytes + kBBytes + kCtlBytes;
// TMEM columns: GEMM accumulator | S (2 buffers) | O | P (2 buffers, bf16 pairs)
constexpr uint32_t kAccCol = 0, kSCol = 64, kOCol = 192, kPCol = 448;

// model geometry the plan is written for (checked by the host)
constexpr int kW = 1024, kHeads = 8, kHD = 256, kQF = kHeads * kHD, kQKV = kQF + 2 * kHD, kMlp = 4096;

// Stage kinds and the static task plan (CTA -> task): consecutive stages use
// mostly disjoint CTAs where a stage is short (attention), so the next
// stage's weights are already in the idle CTAs' rings.
enum Kind : int { K_E = 0, K_QKV = 1, K_ATT = 2, K_O = 3, K_GU = 4, K_DN = 5, K_HEAD = 6 };
constexpr int kPerLayer = 5;
__host__ __device__ constexpr int stages_per_step(int L) { return 2 + kPerLayer * L; }
// QKV: 40 feature tiles of 64 x the whole K (UMMA M = 64, no split)  CTAs [0, 40)
// ATT: 4 query tiles (16 tokens x 8 heads) x kAttSplits KV splits      CTAs [80, 80 + 4 * splits)
// O:   8 x 16 (2 k-blocks)                                             CTAs [0, 80) u [96, 144)
// GU:  128 tiles of 64 x the whole K (M = 64, no split)                CTAs [20, 148)
// DN:  8 x 16 (4 k-blocks)                                             CTAs [0, 128)
// HEAD: 1 x 8 (2 k-blocks)                                             CTAs [128, 136)
#ifndef SF_B1_ATT_SPLITS
#define SF_B1_ATT_SPLITS 7
#endif
constexpr int kAttQT = 4, kAttSplits = SF_B1_ATT_SPLITS;
// split CTAs per output tile (arrival counter modulus)
__device__ __forceinline__ int splits_of(int kind) { return kind == K_HEAD ? 8 : 16; }

__device__ __forceinline__ int task_of(int kind, int c) {
  switch (kind) {
    case K_QKV: return c < 40 ? c : -1;
    case K_ATT: return (c >= 80 && c < 80 + kAttQT * kAttSplits) ? c - 80 : -1;
    case K_O: return c < 80 ? c : ((c >= 96 && c < 144) ? c - 16 : -1);
    case K_GU: return c >= 20 ? c - 20 : -1;
    case K_DN: return c < 128 ? c : -1;
    case K_HEAD: return (c >= 128 && c < 136) ? c - 128 : -1;
    default: return -1;
  }
}

struct Gemm {
  int tile, kb0, items;  // weight tile, first 64-wide k-block, ring items (32 KB each)
  bool m64;              // 64-row tile over the whole K (items of 4 k-blocks), else 128 rows (items of 2)
};

__device__ __forceinline__ Gemm gemm_of(int kind, int t) {
  Gemm g;
  switch (kind) {
    case K_QKV: g.tile = t; g.kb0 = 0; g.items = 4; g.m64 = true; break;
    case K_O: g.tile = t % 8; g.kb0 = (t / 8) * 2; g.items = 1; g.m64 = false; break;
    case K_GU: g.tile = t; g.kb0 = 0; g.items = 4; g.m64 = true; break;
    case K_DN: g.tile = t % 8; g.kb0 = (t / 8) * 4; g.items = 2; g.m64 = false; break;
    default: g.tile = 0; g.kb0 = t * 2; g.items = 1; g.m64 = false; break;  // HEAD
  }
  return g;
}

struct Params {
  CUtensorMap wmap[4 * kMaxL + 1];  // per layer: qkv, o, gu, down; then the head (box 64 x 128, SW128)
  CUtensorMap wmap64[2 * kMaxL];    // per layer: qkv, gu with 64-row boxes (M = 64 tiles)
  CUtensorMap qmap;                 // qb [64 * 8 rows][256] (box 64 x 128)
  CUtensorMap kmap;                 // kb [64 keys][256]     (box 64 x 64)
  CUtensorMap vmap;                 // vt [256 dims][64 keys] (box 64 x 256)
  CUtensorMap xmap;                 // xb [64 rows][1024]     (box 64 x 64): QKV / GU / HEAD operand
  CUtensorMap hmap;                 // hb [64 rows][4096]     (box 64 x 64): DN operand
  CUtensorMap pmap;                 // part_o [4 * splits * 128][256] (box 64 x 128): attention partial store
  int L, T, H, D, S, P, n_steps;
  int npb;                          // prefix key blocks (64 keys)
  int att_b[kAttSplits + 1];        // key-block range of each KV split (the suffix block is index npb)
  float inv_width, eps, scale_log2;
  const uint8_t* k_img;             // [L][E][npb][32 KB] pre-swizzled prefix K blocks
  const uint8_t* v_img;             // same for V^T
  int n_img_envs;
  const int* env_map;               // device: prefix pool slot of the env (null: 0)
  const float2* rope;               // [P + T][128] (cos, sin)
  const float *a_w, *a_b, *s_w, *s_b, *out_b;  // [W][D], [W], [W][S], [W], [D]
  const float* temb;                // [n_steps][W]
  const float* state;               // [S]
  float *x, *acc_qkv, *acc_gu, *acc_head;  // [64][W], [64][2560], [64][8192], [64][D]
  float *ssq1, *ssq2;               // [L + 1][64] (x before QKV of layer l; [L]: before the head), [L][64] (before GU)
  bf16 *qb, *kb, *vt;               // finalised q [64*8][256], k [64][256], v^T [256][64] (pad rows stay 0)
  bf16 *xb, *hb;                    // bf16 residual [64][1024], GeGLU output [64][4096] (pad rows stay 0)
  unsigned* cnt;                    // [8 kinds][64 tiles] split arrival counters (zeroed before the launch)
  float* A;                         // [2][H][D] (A[0] = start, written by the host)
  bf16* part_o;                     // [4 qtiles][splits][128 rows][256] normalised split-KV partials
  float2* part_ml;                  // [4][splits][128] (row max in log2 units, row sum)
  float* chunk_out;                 // [H][D]
  int* status;                      // [2]
  unsigned* bar;                    // grid barrier arrivals (zeroed before the launch)
  unsigned long long* dbg;          // optional [grid][stages][4] %globaltimer stamps
};

// ------------------------------------------------------------ helpers

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void workers_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(sm100::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(sm100::smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(sm100::smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanh_fast(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint4 pack8(const float (&v)[8]) {
  return make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
}
__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
// 16 B unit u (8 bf16) of row r of a SWIZZLE_128B K-major tile (rows of 128 B)
__device__ __forceinline__ uint32_t sw128(int r, int u) { return (uint32_t)(r * 128 + ((u ^ (r & 7)) << 4)); }

__device__ __forceinline__ float rms_scale(const Params& p, const float* ssq, int t) {
  return rsqrtf(__ldcg(ssq + t) * p.inv_width + p.eps);
}

// one worker thread stamps (a same-address store from every thread would
// serialise in L2 and distort the trace)
__device__ __forceinline__ void stamp(const Params& p, int st, int n_st, int k) {
  if (p.dbg && threadIdx.x == 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.dbg[((size_t)blockIdx.x * n_st + st) * 8 + k] = t;
  }
}

// stage index -> (kind, layer, step)
struct StageRef {
  int kind, l, step;
};
__device__ __forceinline__ StageRef stage_ref(const Params& p, int st) {
  const int per = stages_per_step(p.L);
  StageRef r;
  r.step = st / per;
  const int j = st - r.step * per;
  r.l = 0;
  if (j == 0) {
    r.kind = K_E;
  } else if (j == per - 1) {
    r.kind = K_HEAD;
  } else {
    r.l = (j - 1) / kPerLayer;
    r.kind = K_QKV + (j - 1) % kPerLayer;
  }
  return r;
}

__device__ __forceinline__ const CUtensorMap* wmap_of(const Params& p, int kind, int l) {
  switch (kind) {
    case K_QKV: return &p.wmap64[2 * l + 0];
    case K_O: return &p.wmap[4 * l + 1];
    case K_GU: return &p.wmap64[2 * l + 1];
    case K_DN: return &p.wmap[4 * l + 3];
    default: return &p.wmap[4 * p.L];
  }
}

// grid barrier: stage st may start once every CTA arrived for stages < st
__device__ __forceinline__ void grid_wait(const Params& p, int st) {
  const unsigned target = (unsigned)gridDim.x * (unsigned)st;
  if (ld_acquire(p.bar) >= target) return;
  const long long t0 = clock64();
  while (ld_acquire(p.bar) < target) {
    if (clock64() - t0 > (1ll << 33)) {
      printf("sf b1 engine: grid barrier timeout (block %d stage %d)\n", blockIdx.x, st);
      __trap();
    }
  }
}

struct Smem {
  uint8_t* ring;
  uint8_t* B;
  uint64_t* full;     // [kSlots]
  uint64_t* empty;    // [kSlots]
  uint64_t* bfull;    // [8] B operand k-block slot landed (TMA, 1 arrival + bytes)
  uint64_t* bempty;   // [8] B operand k-block slot consumed by the MMAs (TMA-fed slots are reused within a stage)
  uint64_t* bfull_w;  // [2] B operand k-block written by all 256 workers (O: split-KV merge)
  uint64_t* acc_full;
  uint64_t* q_full;   // attention Q landed (TMA)
  uint64_t* s_full;   // [2]
  uint64_t* s_free;   // [2]
  uint64_t* p_full;   // [2]
  uint64_t* pv_done;  // [2]
  uint32_t* tmem_slot;
  int* flag;          // last-arriver broadcast
  float* xm;          // [2 parity][2 half][128] softmax pair exchange
  float* wts;         // [64][kAttSplits] split-KV merge weights
  float* rs;          // [64] RMS row scales of the stage
  float2* rope;       // [64 tokens][32 pairs] RoPE (cos, sin) of the QKV tile, staged during the MMAs
};

__device__ __forceinline__ Smem carve(uint8_t* base) {
  Smem s;
  s.ring = base;
  s.B = base + kRingBytes;
  uint8_t* c = s.B + kBBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(c);
  s.full = bars;
  s.empty = bars + 4;
  s.bfull = bars + 8;
  s.bfull_w = bars + 16;
  s.acc_full = bars + 18;
  s.q_full = bars + 19;
  s.s_full = bars + 20;
  s.s_free = bars + 22;
  s.p_full = bars + 24;
  s.pv_done = bars + 26;
  s.bempty = bars + 28;
  s.tmem_slot = reinterpret_cast<uint32_t*>(bars + 36);
  s.flag = reinterpret_cast<int*>(bars + 37);
  // the float scratch starts after the 38 barrier / slot words (304 B): at
  // c + 256 it overlapped bempty[4..7] and the flag, so the softmax exchange
  // of an attention stage could corrupt a live B-slot barrier
  float* f = reinterpret_cast<float*>(c + 512);
  s.xm = f;            // 512 floats
  s.wts = f + 512;     // 64 * kAttSplits
  s.rs = f + 512 + 64 * kAttSplits;
  s.rope = reinterpret_cast<float2*>(c + 8192);
  return s;
}

// ------------------------------------------------------------ producer (warp 0)

__device__ __forceinline__ void produce(const Params& p, const Smem& sm, int n_st) {
  const uint64_t pol_w = sm100::policy_evict_first();
  const uint64_t pol_kv = sm100::policy_evict_last();
  const int c = blockIdx.x;
  const int slot_env = p.env_map ? __ldg(p.env_map) : 0;
  uint32_t g = 0, bfull_ph = 0, bempty_ph = 0, bused = 0;
  for (int st = 0; st < n_st; ++st) {
    const StageRef r = stage_ref(p, st);
    if (r.step >= p.n_steps) break;
    const int t = task_of(r.kind, c);
    if (t < 0) continue;
    if (r.kind == K_ATT) {
      // ring items K_j, V_j of the split's key blocks: prefix blocks from the
      // pool images (no dependency), the suffix block and Q from this layer's
      // finalised q/k/v (after the grid barrier). The items that fit the ring
      // are issued first, Q next (the MMAs of later items need it).
      const int qt = t % kAttQT, split = t / kAttQT;
      const int jb0 = p.att_b[split], n_items = 2 * (p.att_b[split + 1] - jb0);
      bool q_done = false;
      for (int i = 0; i <= n_items; ++i) {
        if (!q_done && (i == n_items || i >= kSlots || jb0 + (i >> 1) >= p.npb)) {
          grid_wait(p, st);
          fence_async_global();
          sm100::mbar_arrive_expect_tx(sm.q_full, 65536);
          for (int ch = 0; ch < 4; ++ch)
            sm100::tma_load_2d(&p.qmap, sm.q_full, sm.B + ch * 16384, ch * 64, qt * 128, pol_kv);
          q_done = true;
        }
        if (i == n_items) break;
        const int j = jb0 + (i >> 1), part = i & 1;
        const int s = g % kSlots;
        if (g >= kSlots) sm100::mbar_wait(&sm.empty[s], ((g / kSlots) & 1) ^ 1);
        sm100::mbar_arrive_expect_tx(&sm.full[s], kSlotBytes);
        uint8_t* dst = sm.ring + s * kSlotBytes;
        if (j < p.npb) {
          const uint8_t* img = (part ? p.v_img : p.k_img) +
                               (((size_t)r.l * p.n_img_envs + slot_env) * p.npb + j) * kSlotBytes;
          bulk_load(dst, img, kSlotBytes, &sm.full[s], pol_kv);
        } else if (part == 0) {
          for (int ch = 0; ch < 4; ++ch) sm100::tma_load_2d(&p.kmap, &sm.full[s], dst + ch * 8192, ch * 64, 0, pol_kv);
        } else {
          sm100::tma_load_2d(&p.vmap, &sm.full[s], dst, 0, 0, pol_kv);
        }
        ++g;
      }
      continue;
    }
    const Gemm gm = gemm_of(r.kind, t);
    const CUtensorMap* map = wmap_of(p, r.kind, r.l);
    for (int i = 0; i < gm.items; ++i, ++g) {
      const int s = g % kSlots;
      if (g >= kSlots) sm100::mbar_wait(&sm.empty[s], ((g / kSlots) & 1) ^ 1);
      sm100::mbar_arrive_expect_tx(&sm.full[s], kSlotBytes);
      uint8_t* dst = sm.ring + s * kSlotBytes;
      if (gm.m64) {
        for (int sub = 0; sub < 4; ++sub)
          sm100::tma_load_2d(map, &sm.full[s], dst + sub * 8192, (gm.kb0 + 4 * i + sub) * 64, gm.tile * 64, pol_w);
      } else {
        sm100::tma_load_2d(map, &sm.full[s], dst, (gm.kb0 + 2 * i) * 64, gm.tile * 128, pol_w);
        sm100::tma_load_2d(map, &sm.full[s], dst + 16384, (gm.kb0 + 2 * i + 1) * 64, gm.tile * 128, pol_w);
      }
    }
    if (r.kind != K_O) {
      // bf16 activation operand (written by the previous stage's epilogues),
      // streamed through the 8 B slots (the MMAs free a slot per k-block)
      const CUtensorMap* am = r.kind == K_DN ? &p.hmap : &p.xmap;
      const int row0 = r.kind == K_HEAD ? 1 : 0;  // head rows = action tokens 1..H
      grid_wait(p, st);
      fence_async_global();
      const int nkb = (gm.m64 ? 4 : 2) * gm.items;
      for (int kb = 0; kb < nkb; ++kb) {
        const int b = kb & 7;
        if ((bused >> b) & 1) sm100::mbar_wait(&sm.bempty[b], (bempty_ph >> b) & 1), bempty_ph ^= 1u << b;
        bused |= 1u << b;
        sm100::mbar_arrive_expect_tx(&sm.bfull[b], 8192);
        sm100::tma_load_2d(am, &sm.bfull[b], sm.B + b * 8192, (gm.kb0 + kb) * 64, row0, pol_kv);
      }
    }
  }
}

// ------------------------------------------------------------ MMA issuer (warp 1)

__device__ __forceinline__ void mma_issue(const Params& p, const Smem& sm, uint32_t tmem, int n_st) {
  const int c = blockIdx.x;
  const uint32_t ring = sm100::smem_u32(sm.ring);
  const uint32_t bsm = sm100::smem_u32(sm.B);
  const uint32_t idesc_g = sm100::make_idesc_bf16(128, kTok);
  const uint32_t idesc_g64 = sm100::make_idesc_bf16(64, kTok);
  const uint32_t idesc_s = sm100::make_idesc_bf16(128, 64);
  const uint32_t idesc_o = sm100::make_idesc_bf16(128, kHD);
  uint32_t g = 0, nq = 0, ablk = 0, bph = 0, bphw = 0;
  for (int st = 0; st < n_st; ++st) {
    const StageRef r = stage_ref(p, st);
    if (r.step >= p.n_steps) break;
    const int t = task_of(r.kind, c);
    if (t < 0) continue;
    if (r.kind == K_ATT) {
      sm100::mbar_wait(sm.q_full, nq & 1);
      ++nq;
      const int split = t / kAttQT;
      const int nb = p.att_b[split + 1] - p.att_b[split];
      auto issue_pv = [&](int i) {
        const uint32_t blk = ablk + i, pb = blk & 1;
        sm100::mbar_wait(&sm.p_full[pb], (blk >> 1) & 1);
        const uint32_t gv = g + 2 * i + 1, sv = gv % kSlots;
        sm100::mbar_wait(&sm.full[sv], (gv / kSlots) & 1);
        sm100::tc_fence_after();
        const uint32_t v_addr = ring + sv * kSlotBytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // A = P from TMEM: 16 keys = 8 columns per MMA
          sm100::umma_bf16_ts(tmem + kOCol, tmem + kPCol + pb * 32 + kk * 8,
                              sm100::make_sw128_desc(v_addr + kk * 32), idesc_o, (i | kk) != 0);
        sm100::umma_commit(&sm.pv_done[pb]);
        sm100::umma_commit(&sm.empty[sv]);
      };
      for (int i = 0; i < nb; ++i) {
        const uint32_t blk = ablk + i, sb = blk & 1;
        const uint32_t gk = g + 2 * i, sk = gk % kSlots;
        sm100::mbar_wait(&sm.full[sk], (gk / kSlots) & 1);
        if (blk >= 2) sm100::mbar_wait(&sm.s_free[sb], ((blk >> 1) & 1) ^ 1);
        sm100::tc_fence_after();
        const uint32_t k_addr = ring + sk * kSlotBytes;
#pragma unroll
        for (int kk = 0; kk < kHD / 16; ++kk) {
          const int ch = kk >> 2, w = kk & 3;
          sm100::umma_bf16(tmem + kSCol + sb * 64, sm100::make_sw128_desc(bsm + ch * 16384 + w * 32),
                           sm100::make_sw128_desc(k_addr + ch * 8192 + w * 32), idesc_s, kk != 0);
        }
        sm100::umma_commit(&sm.s_full[sb]);
        sm100::umma_commit(&sm.empty[sk]);
        if (i >= 1) issue_pv(i - 1);
      }
      if (nb > 0) issue_pv(nb - 1);
      g += 2 * nb;
      ablk += nb;
      continue;
    }
    const Gemm gm = gemm_of(r.kind, t);
    const bool worker_b = r.kind == K_O;
    const int per = gm.m64 ? 4 : 2;                     // k-blocks per ring item
    const uint32_t a_step = gm.m64 ? 8192 : 16384;      // bytes per weight k-block
    const uint32_t idesc = gm.m64 ? idesc_g64 : idesc_g;
    for (int i = 0; i < gm.items; ++i, ++g) {
      const int s = g % kSlots;
      sm100::mbar_wait(&sm.full[s], (g / kSlots) & 1);
      const uint32_t a_addr = ring + s * kSlotBytes;
      for (int sub = 0; sub < per; ++sub) {
        const int kb = per * i + sub, b = kb & 7;
        if (worker_b) {
          sm100::mbar_wait(&sm.bfull_w[b], (bphw >> b) & 1);
          bphw ^= 1u << b;
        } else {
          sm100::mbar_wait(&sm.bfull[b], (bph >> b) & 1);
          bph ^= 1u << b;
        }
        sm100::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          sm100::umma_bf16(tmem + kAccCol, sm100::make_sw128_desc(a_addr + sub * a_step + kk * 32),
                           sm100::make_sw128_desc(bsm + b * 8192 + kk * 32), idesc, (kb | kk) != 0);
        if (!worker_b) sm100::umma_commit(&sm.bempty[b]);
      }
      sm100::umma_commit(&sm.empty[s]);
    }
    sm100::umma_commit(sm.acc_full);
  }
}

// ------------------------------------------------------------ worker pieces

// O operand = the attention output for features [kb0*64, +128) (one head,
// half of its dims): merge of the kAttSplits normalised bf16 partials with
// weights l_s 2^(m_s - max m) (fixed split order). Thread wt owns units
// idx = wt + 256 k of each k-block (row t = idx >> 3, 16 B unit u = idx & 7).
__device__ __forceinline__ void load_attn_operand(const Params& p, const Smem& sm, int wt, int kb0) {
  const int k0 = kb0 * 64;
  const int h = k0 >> 8, d0 = k0 & 255;
  uint4 raw[2][kAttSplits];
  auto issue = [&](int kb) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int idx = wt + 256 * k, t = idx >> 3, u = idx & 7;
      if (t < p.T) {
        const int qt = t >> 4, r = ((t & 15) << 3) | h;
#pragma unroll
        for (int s = 0; s < kAttSplits; ++s)
          raw[k][s] = __ldcg(reinterpret_cast<const uint4*>(
              p.part_o + ((size_t)(qt * kAttSplits + s) * 128 + r) * kHD + d0 + kb * 64 + u * 8));
      } else {
#pragma unroll
        for (int s = 0; s < kAttSplits; ++s) raw[k][s] = make_uint4(0, 0, 0, 0);
      }
    }
  };
  issue(0);
  if (wt < kTok) {
    const int t = wt;
    float w[kAttSplits];
    float tot = 0.f;
    if (t < p.T) {
      const int qt = t >> 4, r = ((t & 15) << 3) | h;
      float2 ml[kAttSplits];
      float mx = -INFINITY;
#pragma unroll
      for (int s = 0; s < kAttSplits; ++s) {
        ml[s] = __ldcg(p.part_ml + (qt * kAttSplits + s) * 128 + r);
        if (ml[s].y > 0.f) mx = fmaxf(mx, ml[s].x);
      }
#pragma unroll
      for (int s = 0; s < kAttSplits; ++s) {
        w[s] = ml[s].y > 0.f ? ml[s].y * exp2f(ml[s].x - mx) : 0.f;
        tot += w[s];
      }
    } else {
#pragma unroll
      for (int s = 0; s < kAttSplits; ++s) w[s] = 0.f;
    }
    const float inv = tot > 0.f ? 1.f / tot : 0.f;
#pragma unroll
    for (int s = 0; s < kAttSplits; ++s) sm.wts[t * kAttSplits + s] = w[s] * inv;
  }
  workers_bar();
#pragma unroll
  for (int kb = 0; kb < 2; ++kb) {
    if (kb) issue(kb);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int idx = wt + 256 * k, t = idx >> 3, u = idx & 7;
      float o[8];
#pragma unroll
      for (int z = 0; z < 8; ++z) o[z] = 0.f;
#pragma unroll
      for (int s = 0; s < kAttSplits; ++s) {
        const float w = sm.wts[t * kAttSplits + s];
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&raw[k][s]);
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          const float2 f = __bfloat1622float2(b2[z]);
          o[2 * z] = fmaf(w, f.x, o[2 * z]);
          o[2 * z + 1] = fmaf(w, f.y, o[2 * z + 1]);
        }
      }
      *reinterpret_cast<uint4*>(sm.B + kb * 8192 + sw128(t, u)) = pack8(o);
    }
    fence_async_smem();
    sm100::mbar_arrive(&sm.bfull_w[kb]);
  }
}

// Accumulator epilogue: TMEM (128 features x 64 tokens) -> per-warp SMEM
// transpose -> red.global.add.v4.f32 into dst[t][f0 + f] for t < nrows, f < nfeat.
__device__ __forceinline__ void epilogue_red(const Smem& sm, uint32_t tmem, int warp, int lane, float* dst, int ld,
                                             int f0, int nrows, int nfeat) {
  const int q = warp & 3, half = (warp - 2) >> 2;
  uint32_t v[2][16];
  const uint32_t ta = tmem + kAccCol + ((uint32_t)(q * 32) << 16) + half * 32;
  sm100::tmem_ld16(ta, v[0]);
  sm100::tmem_ld16(ta + 16, v[1]);
  sm100::tmem_ld_wait();
  float* stg = reinterpret_cast<float*>(sm.B) + (warp - 2) * 1024;  // [32 tokens][32 features]
#pragma unroll
  for (int j = 0; j < 32; ++j) stg[j * 32 + lane] = __uint_as_float(v[j >> 4][j & 15]);
  __syncwarp();
  const int fq = q * 32 + (lane & 7) * 4;
  if (fq < nfeat) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int tl = (lane >> 3) + 4 * k;
      const int t = half * 32 + tl;
      if (t < nrows) {
        const float4 a = *reinterpret_cast<const float4*>(stg + tl * 32 + (lane & 7) * 4);
        red_add_v4(dst + (size_t)t * ld + f0 + fq, a);
      }
    }
  }
}

// ---- residual tile epilogue (units of 8 outputs)

// rows [r0, r0 + nr) of residual tile f (nr * 16 <= kWorkers): the share of
// one split CTA once every split of the tile has reduced into L2
__device__ __forceinline__ void tile_epi_resid_rows(const Params& p, int wt, int f, int r0, int nr,
                                                    float* ssq_out) {
  if (wt >= nr * 16) return;
  const int t = r0 + (wt >> 4), u = wt & 15;  // 16 lanes per row (half a warp)
  float v[8];
  float sq = 0.f;
  if (t < p.T) {
    const float* src = p.x + (size_t)t * kW + f * 128 + u * 8;
    const float4 a = ldcg4(src), b = ldcg4(src + 4);
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
#pragma unroll
    for (int k = 0; k < 8; ++k) sq = fmaf(v[k], v[k], sq);
    __stcg(reinterpret_cast<uint4*>(p.xb + (size_t)t * kW + f * 128 + u * 8), pack8(v));
  }
  // the 16 lanes of the row are one half-warp: all of them reach the shuffles
  const unsigned hm = (wt & 16) ? 0xffff0000u : 0x0000ffffu;
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) sq += __shfl_xor_sync(hm, sq, off);
  if (u == 0 && t < p.T) atomicAdd(ssq_out + t, sq);
}

// ---- M = 64 accumulators (QKV, gate/up: whole K in one CTA, no split):
// feature row 16 q + l of the tile sits in TMEM lane 32 q + l (l < 16) of
// lane quarter q; columns are tokens. The epilogue runs in the CTA itself.

__device__ __forceinline__ void acc64_load(uint32_t tmem, int warp, uint32_t (&v)[2][16]) {
  const int q = warp & 3, half = (warp - 2) >> 2;
  const uint32_t ta = tmem + kAccCol + ((uint32_t)(q * 32) << 16) + half * 32;
  sm100::tmem_ld16(ta, v[0]);
  sm100::tmem_ld16(ta + 16, v[1]);
  sm100::tmem_ld_wait();
}

// QKV tile (64 features): q/k = bf16(rope(acc r)) with RoPE pairs (i, i+128)
// on adjacent rows (EPI_QKV's math) -> qb / kb rows; V -> v^T rows.
__device__ __forceinline__ void epi64_qkv(const Params& p, const Smem& sm, uint32_t tmem, int warp, int lane,
                                          int wt, int tile, int st, int n_st) {
  const int q = warp & 3, half = (warp - 2) >> 2;
  uint32_t v[2][16];
  acc64_load(tmem, warp, v);
  stamp(p, st, n_st, 4);
  const int fl = 16 * q + (lane & 15);
  const int n = tile * 64 + fl;
  if (tile < 36) {
    const int i = (n & 255) >> 1, second = n & 1;
    const int col = (i & 31) + 32 * second;
    bf16* stg = reinterpret_cast<bf16*>(sm.B);  // [64 tokens][64]: dims i0 + [0, 32) | 128 + i0 + [0, 32)
#pragma unroll
    for (int j0 = 0; j0 < 32; j0 += 16) {
      float2 cs[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) cs[k] = sm.rope[(half * 32 + j0 + k) * 32 + (fl >> 1)];
      float yv[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int j = j0 + k, tok = half * 32 + j;
        const float x = __uint_as_float(v[j >> 4][j & 15]) * sm.rs[tok];
        const float partner = __shfl_xor_sync(0xffffffffu, x, 1);
        const float a = second ? partner : x, b = second ? x : partner;
        yv[k] = second ? (b * cs[k].x + a * cs[k].y) : (a * cs[k].x - b * cs[k].y);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (lane < 16) stg[(half * 32 + j0 + k) * 64 + col] = __float2bfloat16_rn(yv[k]);
    }
    stamp(p, st, n_st, 5);
    workers_bar();
    stamp(p, st, n_st, 1);
    const int h = tile >> 2, i0 = (tile & 3) * 32;
    for (int idx = wt; idx < p.T * 8; idx += kWorkers) {
      const int tok = idx >> 3, u = idx & 7;
      const uint4 val = *reinterpret_cast<const uint4*>(stg + tok * 64 + 8 * u);
      const int dim = u < 4 ? i0 + 8 * u : 128 + i0 + 8 * (u - 4);
      bf16* dst = h < kHeads ? p.qb + ((size_t)tok * kHeads + h) * kHD : p.kb + (size_t)tok * kHD;
      __stcg(reinterpret_cast<uint4*>(dst + dim), val);
    }
  } else if (lane < 16) {
    const int d = n - kQF - kHD;
#pragma unroll
    for (int c8 = 0; c8 < 4; ++c8) {
      float f[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = 8 * c8 + k;
        f[k] = __uint_as_float(v[j >> 4][j & 15]) * sm.rs[half * 32 + j];
      }
      __stcg(reinterpret_cast<uint4*>(p.vt + (size_t)d * kTok + half * 32 + 8 * c8), pack8(f));
    }
  }
}

// gate/up tile (64 interleaved rows = 32 h columns): h = bf16(gelu_tanh(g r) * (u r))
__device__ __forceinline__ void epi64_geglu(const Params& p, const Smem& sm, uint32_t tmem, int warp, int lane,
                                            int wt, int tile, int st, int n_st) {
  const int q = warp & 3, half = (warp - 2) >> 2;
  uint32_t v[2][16];
  acc64_load(tmem, warp, v);
  stamp(p, st, n_st, 4);
  const int fl = 16 * q + (lane & 15);
  bf16* stg = reinterpret_cast<bf16*>(sm.B);  // [64 tokens][32 h]
  // branch-free body (a per-iteration branch serialises the unrolled loop)
  const bool writer = lane < 16 && !(lane & 1);
#pragma unroll
  for (int j0 = 0; j0 < 32; j0 += 16) {
    float hv[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int j = j0 + k;
      const float x = __uint_as_float(v[j >> 4][j & 15]) * sm.rs[half * 32 + j];
      const float partner = __shfl_xor_sync(0xffffffffu, x, 1);
      hv[k] = gelu_tanh(x) * partner;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (writer) stg[(half * 32 + j0 + k) * 32 + (fl >> 1)] = __float2bfloat16_rn(hv[k]);
  }
  stamp(p, st, n_st, 5);
  workers_bar();
  stamp(p, st, n_st, 1);
  for (int idx = wt; idx < p.T * 4; idx += kWorkers) {
    const int tok = idx >> 2, u = idx & 3;
    __stcg(reinterpret_cast<uint4*>(p.hb + (size_t)tok * kMlp + tile * 32 + 8 * u),
           *reinterpret_cast<const uint4*>(stg + tok * 32 + 8 * u));
  }
}

// ------------------------------------------------------------ the kernel

__global__ void __launch_bounds__(kThreads, 1) engine_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the __shared__ array (a round trip through
  // uintptr_t would make every SMEM access below a generic LD/ST)
  uint8_t* base = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  const Smem sm = carve(base);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_st = stages_per_step(p.L) * p.n_steps + 1;
  const int c = blockIdx.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      sm100::mbar_init(&sm.full[s], 1);
      sm100::mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 8; ++b) {
      sm100::mbar_init(&sm.bfull[b], 1);
      sm100::mbar_init(&sm.bempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) sm100::mbar_init(&sm.bfull_w[b], kWorkers);
    sm100::mbar_init(sm.acc_full, 1);
    sm100::mbar_init(sm.q_full, 1);
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&sm.s_full[b], 1);
      sm100::mbar_init(&sm.s_free[b], kWorkers);
      sm100::mbar_init(&sm.p_full[b], kWorkers);
      sm100::mbar_init(&sm.pv_done[b], 1);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<512>(sm.tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *sm.tmem_slot;

  if (warp == 0) {
    if (sm100::elect_one()) {
      for (int i = 0; i <= 4 * p.L; ++i) sm100::tma_prefetch_desc(&p.wmap[i]);
      sm100::tma_prefetch_desc(&p.qmap);
      sm100::tma_prefetch_desc(&p.kmap);
      sm100::tma_prefetch_desc(&p.vmap);
      sm100::tma_prefetch_desc(&p.xmap);
      sm100::tma_prefetch_desc(&p.hmap);
      produce(p, sm, n_st);
    }
    __syncwarp();
  } else if (warp == 1) {
    if (sm100::elect_one()) mma_issue(p, sm, tmem, n_st);
    __syncwarp();
  } else {
    // ------------------------------------------------------------ workers
    const int wt = threadIdx.x - 64;
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int HD_ = p.H * p.D;
    const int gid = c * kWorkers + wt, gstride = gridDim.x * kWorkers;
    uint32_t nacc = 0, ablk = 0;
    float* A_new = reinterpret_cast<float*>(sm.B);  // E stage scratch [H][D]
    for (int st = 0; st < n_st; ++st) {
      const StageRef r = stage_ref(p, st);
      if (st > 0) {
        if (wt == 0) grid_wait(p, st);
        workers_bar();
      }
      stamp(p, st, n_st, 0);
      const int t = task_of(r.kind, c);
      if (t >= 0 && (r.kind == K_QKV || r.kind == K_GU)) {
        if (wt < kTok) {
          const float* ssq = (r.kind == K_QKV ? p.ssq1 : p.ssq2) + r.l * kTok;
          sm.rs[wt] = wt < p.T ? rsqrtf(__ldcg(ssq + wt) * p.inv_width + p.eps) : 0.f;
        }
        if (r.kind == K_QKV && t < 36) {
          // the tile's 32 RoPE pairs for every token, staged while the MMAs
          // run (the epilogue's L2 table loads were on the critical path)
          const int i_base = ((t * 64) & 255) >> 1;
          for (int e = wt; e < kTok * 32; e += kWorkers) {
            const int tok = e >> 5, j = e & 31;
            sm.rope[e] = tok < p.T ? __ldg(p.rope + (size_t)(p.P + tok) * 128 + i_base + j) : make_float2(1.f, 0.f);
          }
        }
      }
      if (r.kind == K_E) {
        // ---- Euler update of the previous step (flowpolicy.py:289-291) + embedding
        const int i = r.step;
        // this CTA's embedding rows (features 8c .. 8c + 7: action / state
        // weights, biases, time embedding) and the state go to SMEM first, in
        // parallel with the Euler update's loads: the embedding's dependent
        // global-load chains held the stage ~5 us
        float* e_aw = reinterpret_cast<float*>(sm.rope);  // [8][D] | [8][S] | a_b[8] | s_b[8] | temb[8] | state[S]
        float* e_sw = e_aw + 8 * p.D;
        float* e_ab = e_sw + 8 * p.S;
        float* e_sb = e_ab + 8;
        float* e_te = e_sb + 8;
        float* e_st = e_te + 8;
        if (i < p.n_steps && c < kW / 8) {
          for (int e = wt; e < 8 * p.D; e += kWorkers) e_aw[e] = __ldg(p.a_w + (size_t)c * 8 * p.D + e);
          for (int e = wt; e < 8 * p.S; e += kWorkers) e_sw[e] = __ldg(p.s_w + (size_t)c * 8 * p.S + e);
          if (wt < 8) {
            e_ab[wt] = __ldg(p.a_b + c * 8 + wt);
            e_sb[wt] = __ldg(p.s_b + c * 8 + wt);
            e_te[wt] = __ldg(p.temb + (size_t)i * kW + c * 8 + wt);
          }
          if (wt < p.S) e_st[wt] = __ldg(p.state + wt);
        }
        if (i > 0) {
          const float* Aprev = p.A + ((i - 1) & 1) * HD_;
          const float* ssqf = p.ssq1 + (size_t)p.L * kTok;
          for (int e0 = wt; e0 < HD_; e0 += 8 * kWorkers) {  // one round of loads (H * D <= 2048)
            float hv[8], ap[8], rf[8];
#pragma unroll
            for (int z = 0; z < 8; ++z) {
              const int e = e0 + z * kWorkers;
              if (e < HD_) {
                hv[z] = __ldcg(p.acc_head + e);
                ap[z] = __ldcg(Aprev + e);
                rf[z] = __ldcg(ssqf + 1 + e / p.D);  // row h of the head = token h + 1
              }
            }
#pragma unroll
            for (int z = 0; z < 8; ++z) {
              const int e = e0 + z * kWorkers;
              if (e >= HD_) continue;
              const int d = e % p.D;
              const float v = hv[z] * rsqrtf(rf[z] * p.inv_width + p.eps) + __ldg(p.out_b + d);
              const float nxt = __fadd_rn(ap[z], __fdiv_rn(v, (float)p.n_steps));
              A_new[e] = nxt;
              if (c == 0) {
                if (i < p.n_steps) __stcg(p.A + (i & 1) * HD_ + e, nxt);
                else p.chunk_out[e] = nxt;
                if (!isfinite(v)) atomicCAS(&p.status[1], 0, 1);
                if (!isfinite(nxt)) atomicCAS(&p.status[0], -1, i - 1);
              }
            }
          }
        } else {
          for (int e = wt; e < HD_; e += kWorkers) A_new[e] = __ldcg(p.A + e);
          if (c == 0 && wt == 0) {
            p.status[0] = -1;
            p.status[1] = 0;
          }
        }
        workers_bar();
        if (i < p.n_steps) {
          if (c < kW / 8) {
            // features n = 8c + (wt & 7), tokens wt >> 3 and +32 (embed_kernel's
            // FMA order); x fp32 + its bf16 copy + the first RMSNorm's sums
            const int n = c * 8 + (wt & 7), nl = wt & 7;
            const float temb = e_te[nl];
            for (int tk0 = 0; tk0 < 64; tk0 += 32) {
              const int tk = tk0 + (wt >> 3);
              float v = 0.f;
              if (tk == 0) {
                v = e_sb[nl];
                for (int cc = 0; cc < p.S; ++cc) v = fmaf(e_sw[nl * p.S + cc], e_st[cc], v);
              } else if (tk < p.T) {
                v = e_ab[nl];
                const float* arow = A_new + (tk - 1) * p.D;
                const float* wrow = e_aw + nl * p.D;
                for (int c4 = 0; c4 < p.D / 4; ++c4) {
                  v = fmaf(wrow[4 * c4], arow[4 * c4], v);
                  v = fmaf(wrow[4 * c4 + 1], arow[4 * c4 + 1], v);
                  v = fmaf(wrow[4 * c4 + 2], arow[4 * c4 + 2], v);
                  v = fmaf(wrow[4 * c4 + 3], arow[4 * c4 + 3], v);
                }
                v = v + temb;
              }
              float sq = v * v;
              sq += __shfl_xor_sync(0xffffffffu, sq, 1);
              sq += __shfl_xor_sync(0xffffffffu, sq, 2);
              sq += __shfl_xor_sync(0xffffffffu, sq, 4);
              if (tk < p.T) {
                __stcg(p.x + (size_t)tk * kW + n, v);
                p.xb[(size_t)tk * kW + n] = __float2bfloat16_rn(v);
                if ((wt & 7) == 0) atomicAdd(p.ssq1 + tk, sq);
              }
            }
          }
          // chores: this step's other RMS sums start at zero
          for (int i2 = gid; i2 < (2 * p.L - 1) * kTok; i2 += gstride) {
            if (i2 < (p.L - 1) * kTok) p.ssq1[kTok + i2] = 0.f;
            else p.ssq2[i2 - (p.L - 1) * kTok] = 0.f;
          }
        }
      } else if (t >= 0 && r.kind == K_ATT) {
        // ---- attention task: (query tile, KV split); Q / K / V come by TMA
        const int qt = t % kAttQT, split = t / kAttQT;
        const int jb0 = p.att_b[split], nb = p.att_b[split + 1] - jb0;
        const int rr = q * 32 + lane;  // query row == TMEM lane
        const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
        const int tok = qt * 16 + (rr >> 3);
        const bool real = tok < p.T;
        float m_used = -INFINITY, l_sum = 0.f;
        for (int i = 0; i < nb; ++i) {
          const int j = jb0 + i;
          const uint32_t blk = ablk + i, s = blk & 1;
          sm100::mbar_wait(&sm.s_full[s], (blk >> 1) & 1);
          if (i == 0) stamp(p, st, n_st, 1);
          sm100::tc_fence_after();
          uint32_t raw[2][16];
          sm100::tmem_ld16(t_lane + kSCol + s * 64 + half * 32, raw[0]);
          sm100::tmem_ld16(t_lane + kSCol + s * 64 + half * 32 + 16, raw[1]);
          sm100::tmem_ld_wait();
          sm100::tc_fence_before();
          sm100::mbar_arrive(&sm.s_free[s]);
          int lo = 0, hi;
          if (!real) hi = 0;
          else if (j < p.npb) hi = p.P - j * 64;
          else hi = tok >= 1 ? p.T : 1;  // state token: prefix + itself
          lo -= half * 32;
          hi -= half * 32;
          float sv[32];
          float mb = -INFINITY;
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) {
            const float x = __uint_as_float(raw[cc >> 4][cc & 15]);
            sv[cc] = (cc >= lo && cc < hi) ? x : -INFINITY;
            mb = fmaxf(mb, sv[cc]);
          }
          sm.xm[(s * 2 + half) * 128 + rr] = mb;
          asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
          mb = fmaxf(sm.xm[(s * 2) * 128 + rr], sm.xm[(s * 2 + 1) * 128 + rr]) * p.scale_log2;
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
            pw[k] = pack2(p0, p1);
          }
          if (i >= 1) {
            const uint32_t pb = (blk - 1) & 1;
            sm100::mbar_wait(&sm.pv_done[pb], ((blk - 1) >> 1) & 1);
            sm100::tc_fence_after();
          }
          const bool any_rescale = __any_sync(0xffffffffu, rescale);
          if (any_rescale && i >= 1) {
            l_sum *= alpha;
#pragma unroll 1
            for (int c0 = half * 128; c0 < half * 128 + 128; c0 += 16) {
              uint32_t o[16];
              sm100::tmem_ld16(t_lane + kOCol + c0, o);
              sm100::tmem_ld_wait();
#pragma unroll
              for (int k = 0; k < 16; ++k) o[k] = __float_as_uint(__uint_as_float(o[k]) * alpha);
              sm100::tmem_st16(t_lane + kOCol + c0, o);
            }
            sm100::tmem_st_wait();
          } else if (rescale) {
            l_sum *= alpha;
          }
          l_sum += lp;
          sm100::tmem_st16(t_lane + kPCol + s * 32 + half * 16, pw);
          sm100::tmem_st_wait();
          sm100::tc_fence_before();
          sm100::mbar_arrive(&sm.p_full[s]);
        }
        if (nb > 0) {
          const uint32_t lb = ablk + nb - 1;
          sm100::mbar_wait(&sm.pv_done[lb & 1], (lb >> 1) & 1);
          sm100::tc_fence_after();
        }
        {
          const int ps = (ablk + nb) & 1;
          sm.xm[(ps * 2 + half) * 128 + rr] = l_sum;
          asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
          l_sum = sm.xm[(ps * 2) * 128 + rr] + sm.xm[(ps * 2 + 1) * 128 + rr];
        }
        stamp(p, st, n_st, 2);
        // normalised bf16 partial (SW128 chunks in the now free Q region, one
        // TMA store of 64 KB) + (m, l) of this split
        const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          uint32_t o[4][16];
#pragma unroll
          for (int u = 0; u < 4; ++u) sm100::tmem_ld16(t_lane + kOCol + half * 128 + c2 * 64 + 16 * u, o[u]);
          sm100::tmem_ld_wait();
          uint8_t* chunk = sm.B + (half * 2 + c2) * 16384;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            float f[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) f[k] = __uint_as_float(o[u >> 1][8 * (u & 1) + k]) * inv;
            *reinterpret_cast<uint4*>(chunk + sw128(rr, u)) = pack8(f);
          }
        }
        if (half == 0)
          __stcg(p.part_ml + (qt * kAttSplits + split) * 128 + rr, make_float2(m_used, l_sum));
        fence_async_smem();
        sm100::tc_fence_before();
        workers_bar();
        if (wt == 0) {
          const int row0 = (qt * kAttSplits + split) * 128;
          for (int ch = 0; ch < 4; ++ch) tma_store_2d(&p.pmap, sm.B + ch * 16384, ch * 64, row0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          fence_async_global();
        }
        ablk += nb;
      } else if (t >= 0 && r.kind == K_O) {
        load_attn_operand(p, sm, wt, gemm_of(r.kind, t).kb0);
        stamp(p, st, n_st, 1);
      }
      // ---- chores (zeroing) while the MMAs run: the accumulator's last reader
      // finished >= 1 barrier ago, its next writer starts >= 1 barrier later
      if (r.kind == K_QKV) {
        if (r.l == 0) {
          for (int i2 = gid; i2 < kTok * p.D; i2 += gstride) p.acc_head[i2] = 0.f;
          for (int i2 = gid; i2 < kTok; i2 += gstride) p.ssq1[(size_t)p.L * kTok + i2] = 0.f;
        }
      } else if (r.kind == K_HEAD) {
        for (int i2 = gid; i2 < kTok; i2 += gstride) p.ssq1[i2] = 0.f;
      }
      if (t >= 0 && r.kind != K_ATT && r.kind != K_E) {
        const Gemm gm = gemm_of(r.kind, t);
        sm100::mbar_wait(sm.acc_full, nacc & 1);
        ++nacc;
        sm100::tc_fence_after();
        stamp(p, st, n_st, 2);
        if (gm.m64) {
          workers_bar();  // row scales visible
          stamp(p, st, n_st, 6);
          if (r.kind == K_QKV) epi64_qkv(p, sm, tmem, warp, lane, wt, gm.tile, st, n_st);
          else epi64_geglu(p, sm, tmem, warp, lane, wt, gm.tile, st, n_st);
          sm100::tc_fence_before();
        } else {
        float* dst;
        int ld, nrows = p.T, nfeat = 128;
        if (r.kind == K_HEAD) dst = p.acc_head, ld = p.D, nrows = p.H, nfeat = p.D;
        else dst = p.x, ld = kW;  // O, DOWN: residual
        epilogue_red(sm, tmem, warp, lane, dst, ld, gm.tile * 128, nrows, nfeat);
        sm100::tc_fence_before();
        if (r.kind != K_HEAD) {
          // all split CTAs of the tile finish it together from the L2 sums,
          // 1/S of its rows each, once the last split arrived (a single
          // last-arriver converting the whole tile held the O / down stages
          // ~2 us longer, profiles/r2 engine traces)
          workers_bar();
          const int S = splits_of(r.kind);
          if (wt == 0) {
            unsigned* cp = p.cnt + r.kind * 64 + gm.tile;
            const unsigned target = (atom_add_acq_rel(cp, 1u) / S + 1) * S;
            if (ld_acquire(cp) < target) {
              const long long t0 = clock64();
              while (ld_acquire(cp) < target) {
                if (clock64() - t0 > (1ll << 33)) {
                  printf("sf b1 engine: tile counter timeout (block %d stage %d)\n", blockIdx.x, st);
                  __trap();
                }
              }
            }
          }
          workers_bar();
          const int rows = kTok / S, r0 = (t / 8) * rows;  // task t = split * 8 + tile
          tile_epi_resid_rows(p, wt, gm.tile, r0, rows, r.kind == K_O ? p.ssq2 + r.l * kTok
                                                                      : p.ssq1 + (r.l + 1) * kTok);
        }
        }
      }
      // ---- stage done: every worker's global writes precede the release
      workers_bar();
      stamp(p, st, n_st, 3);
      if (wt == 0 && st + 1 < n_st) red_release_add(p.bar, 1u);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (warp == 1) sm100::tmem_dealloc<512>(tmem);
}

}  // namespace b1
}  // namespace sf
