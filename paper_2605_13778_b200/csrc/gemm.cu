// Host side of the tcgen05 GEMMs: tensor maps, planning (swap-AB + cluster
// split-K for batch-1 shapes, persistent tiles for batched shapes), PDL /
// cluster launch, and a debug C entry point used by the GEMM unit tests.

#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "gemm.cuh"
#include "gemm_host.h"
#include "specflow_b200_internal.h"

namespace sf {
namespace gemm {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

using KernelFn = void (*)(CUtensorMap, CUtensorMap, Params);

template <int KIND>
KernelFn swap_fn() {
  return gemm_swap_kernel<KIND>;
}
template <int KIND>
KernelFn persistent_fn() {
  return gemm_persistent_kernel<KIND>;
}
template <int KIND>
KernelFn pair_fn() {
  return gemm_pair_kernel<KIND>;
}

KernelFn pick_pair(int kind) {
  switch (kind) {
    case EPI_F32: return pair_fn<EPI_F32>();
    case EPI_BF16: return pair_fn<EPI_BF16>();
    case EPI_QKV: return pair_fn<EPI_QKV>();
    case EPI_RESID: return pair_fn<EPI_RESID>();
    case EPI_GEGLU: return pair_fn<EPI_GEGLU>();
    case EPI_TANH_BF16: return pair_fn<EPI_TANH_BF16>();
  }
  return nullptr;
}

KernelFn pick(int kind, bool swap) {
  switch (kind) {
    case EPI_F32: return swap ? swap_fn<EPI_F32>() : persistent_fn<EPI_F32>();
    case EPI_BF16: return swap ? swap_fn<EPI_BF16>() : persistent_fn<EPI_BF16>();
    case EPI_QKV: return swap ? swap_fn<EPI_QKV>() : persistent_fn<EPI_QKV>();
    case EPI_RESID: return swap ? swap_fn<EPI_RESID>() : persistent_fn<EPI_RESID>();
    case EPI_GEGLU: return swap ? swap_fn<EPI_GEGLU>() : persistent_fn<EPI_GEGLU>();
    case EPI_TANH_BF16: return swap ? swap_fn<EPI_TANH_BF16>() : persistent_fn<EPI_TANH_BF16>();
  }
  return nullptr;
}
}  // namespace

int make_map(CUtensorMap* m, const void* ptr, int rows, int K, int ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SF_ECUDA;
  }
  SF_REQUIRE(((uintptr_t)ptr & 15) == 0 && (ld * 2) % 16 == 0, "TMA operand must be 16 B aligned");
  SF_REQUIRE(box_rows >= 1 && box_rows <= 256, "bad TMA box");
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%d K=%d ld=%d box=%d", (int)r, rows, K, ld,
              box_rows);
    return SF_ECUDA;
  }
  return SF_OK;
}

int auto_splits(int tiles, int num_kb) {
  int s = num_sms() / (tiles > 0 ? tiles : 1);
  // portable cluster sizes: 16-CTA clusters cannot all be co-resident (only
  // ~7 fit on the GPCs at once, measured), which doubles the wave count
  if (s > 8) s = 8;
  if (s > num_kb) s = num_kb;
  return s < 1 ? 1 : s;
}

int plan(Op* op, const void* A, int rows_a, int lda, const void* B, int rows_b, int ldb, int K,
         int bn, int splits, int swap_ab, const EpiArgs& e, int max_stages) {
  SF_REQUIRE(bn >= 16 && bn <= 256 && bn % 16 == 0, "bn must be a multiple of 16 in [16, 256]");
  SF_REQUIRE(K % BK == 0, "K (%d) must be a multiple of %d", K, BK);
  SF_REQUIRE(e.kind >= 0 && e.kind < EPI_KINDS, "bad epilogue kind");
  SF_REQUIRE(e.kind != EPI_RESID || swap_ab || bn % 128 == 0, "residual epilogue needs bn %% 128 == 0");
  SF_REQUIRE(swap_ab || rows_a > 0, "empty GEMM");
  Params& p = op->p;
  p = Params{};
  p.rows_a = rows_a;
  p.rows_b = rows_b;
  p.K = K;
  p.bn = bn;
  p.num_kb = K / BK;
  p.swap_ab = swap_ab;
  p.tiles_a = (rows_a + BM - 1) / BM;
  p.tiles_b = (rows_b + bn - 1) / bn;
  p.total_tiles = p.tiles_a * p.tiles_b;
  if (!swap_ab) splits = 1;  // the persistent kernel walks whole-K tiles
  if (splits <= 0) splits = auto_splits(p.total_tiles, p.num_kb);
  splits = splits < 1 ? 1 : (splits > p.num_kb ? p.num_kb : splits);
  SF_REQUIRE(splits <= kMaxSplits, "at most %d K splits", kMaxSplits);
  p.kb_per_split = (p.num_kb + splits - 1) / splits;
  p.splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;  // every split gets >= 1 block
  p.e = e;
  const uint32_t stage_bytes = kAStageBytes + ((bn * BK * 2 + 1023) & ~1023);
  const size_t budget = 227 * 1024 - kTailBytes - 1024;
  int stages = (int)(budget / stage_bytes);
  if (stages > max_stages) stages = max_stages;
  if (stages > 16) stages = 16;
  if (swap_ab && stages > p.kb_per_split) stages = p.kb_per_split < 2 ? 2 : p.kb_per_split;
  SF_REQUIRE(stages >= 2, "GEMM tile does not fit in shared memory");
  p.stages = stages;
  size_t region = (size_t)stages * stage_bytes;
  region = (region + 1023) & ~size_t(1023);
  // split-K partial workspace (caller provides op->p.ws of op->ws_bytes)
  op->ws_bytes = p.splits > 1 ? (size_t)p.splits * p.total_tiles * (bn / 16) * BM * 16 * 4 : 0;
  SF_REQUIRE(region + kTailBytes + 1024 <= 227 * 1024, "GEMM shared memory over budget");
  p.smem_stage_region = (uint32_t)region;
  op->smem = region + kTailBytes + 1024;
  if (swap_ab) {
    op->grid = dim3(p.tiles_a, p.tiles_b, p.splits);
    op->cluster = p.splits;
  } else {
    const int ctas = p.total_tiles < num_sms() ? p.total_tiles : num_sms();
    op->grid = dim3(ctas, 1, 1);
    op->cluster = 1;
  }
  op->fn = reinterpret_cast<void*>(pick(e.kind, swap_ab));
  op->pair = false;
  // batched shapes with whole 256-wide feature tiles run on 2-SM CTA pairs
  // (gemm_pair_kernel): 256 x 256 tiles, half of A and B per SM
  if (!swap_ab && bn == 256 && rows_a >= 4 * 256 && getenv("SF_NO_PAIR") == nullptr) {
    p.tiles_a = (rows_a + 255) / 256;
    p.tiles_b = (rows_b + 255) / 256;
    p.total_tiles = p.tiles_a * p.tiles_b;
    const size_t budget2 = 227 * 1024 - kTailBytes - 1024;
    int st = (int)(budget2 / kPairStageBytes);
    st = st > 16 ? 16 : st;
    p.stages = st;
    p.smem_stage_region = (uint32_t)((size_t)st * kPairStageBytes);
    op->smem = p.smem_stage_region + kTailBytes + 1024;
    int pairs = num_sms() / 2;
    pairs = p.total_tiles < pairs ? p.total_tiles : pairs;
    op->grid = dim3(2 * pairs, 1, 1);
    op->cluster = 2;
    op->pair = true;
    op->fn = reinterpret_cast<void*>(pick_pair(e.kind));
    int rc = make_map(&op->ta, A, rows_a, K, lda, BM);
    if (rc) return rc;
    return make_map(&op->tb, B, rows_b, K, ldb, BM);
  }
  int rc = make_map(&op->ta, A, rows_a, K, lda, BM);
  if (rc) return rc;
  return make_map(&op->tb, B, rows_b, K, ldb, bn);
}

int launch(const Op& op, cudaStream_t stream, bool pdl) {
  SF_REQUIRE(op.ws_bytes == 0 || op.p.ws, "split-K GEMM launched without a workspace");
  static bool attr_done[3 * EPI_KINDS] = {};
  const int slot = op.p.e.kind * 3 + (op.pair ? 2 : op.p.swap_ab ? 1 : 0);
  KernelFn fn = reinterpret_cast<KernelFn>(op.fn);
  if (!attr_done[slot]) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    SF_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_done[slot] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = op.grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = op.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[na].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  ++na;
  if (op.cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = op.pair ? 2 : 1;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = op.pair ? 1 : op.cluster;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  SF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, fn, op.ta, op.tb, op.p));
  count_launch();
  return SF_OK;
}

}  // namespace gemm
}  // namespace sf

namespace {
// Debug entry points own a temporary split-K workspace.
struct DbgWs {
  float* p = nullptr;
  ~DbgWs() {
    if (p) cudaFree(p);
  }
};
int attach_ws(sf::gemm::Op& op, DbgWs& w) {
  if (op.ws_bytes) {
    SF_CHECK_CUDA(cudaMalloc(&w.p, op.ws_bytes));
    op.p.ws = w.p;
  }
  return SF_OK;
}
}  // namespace

// Debug entry: D = A @ B^T with an F32 / BF16 epilogue (optional RMS row
// scale from ssq partials). Synchronises `stream`; not for the hot path.
extern "C" int sf_dbg_gemm(const void* A, int rows_a, const void* B, int rows_b, int K, int bn,
                           int splits, int swap_ab, int epi_kind, void* out, int ld_out,
                           int M_valid, int N_valid, const float* ssq, int ssq_groups, int ssq_ld,
                           float inv_width, void* stream) {
  using namespace sf::gemm;
  SF_REQUIRE(epi_kind == EPI_F32 || epi_kind == EPI_BF16, "debug GEMM supports F32/BF16 epilogues");
  EpiArgs e{};
  e.kind = epi_kind;
  e.M = M_valid;
  e.N = N_valid;
  e.out_f32 = static_cast<float*>(out);
  e.ld_f32 = ld_out;
  e.out_bf16 = static_cast<__nv_bfloat16*>(out);
  e.ld_bf16 = ld_out;
  e.ssq_in = ssq;
  e.ssq_groups = ssq_groups;
  e.ssq_ld = ssq_ld;
  e.inv_width = inv_width;
  e.eps = 1e-6f;
  Op op;
  int rc = plan(&op, A, rows_a, K, B, rows_b, K, K, bn, splits, swap_ab, e);
  DbgWs dws;
  if (!rc) rc = attach_ws(op, dws);
  if (!rc) rc = launch(op, (cudaStream_t)stream, false);
  SF_CHECK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return rc;
}

// Debug timeline: %globaltimer stamps (ns) of CTA (0,0,0) of one warm launch
// of a swap GEMM: 0 entry, 1 prologue done, 2 producer issued all, 3 MMA
// committed, 4 epilogue row scales ready, 5 accumulator ready, 6 partial
// staged, 7 cluster sync, 8 reduce+epilogue done, 9 cluster sync, 10 epilogue
// end, 11 TMEM freed. stamps[12] = host-visible copy (0 = not reached).
extern "C" int sf_dbg_gemm_trace(const void* A, int rows_a, const void* B, int rows_b, int K,
                                 int bn, int splits, void* out, unsigned long long* stamps,
                                 void* stream) {
  using namespace sf::gemm;
  EpiArgs e{};
  e.kind = EPI_F32;
  e.M = rows_b;
  e.N = rows_a;
  e.out_f32 = static_cast<float*>(out);
  e.ld_f32 = e.N;
  e.inv_width = 1.f;
  e.eps = 1e-6f;
  Op op;
  int rc = plan(&op, A, rows_a, K, B, rows_b, K, K, bn, splits, 1, e);
  DbgWs dws;
  if (!rc) rc = attach_ws(op, dws);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  for (int i = 0; i < 3; ++i)
    if ((rc = launch(op, s, false))) return rc;
  unsigned long long* d = nullptr;
  SF_CHECK_CUDA(cudaMalloc(&d, 16 * sizeof(unsigned long long)));
  SF_CHECK_CUDA(cudaMemsetAsync(d, 0, 16 * sizeof(unsigned long long), s));
  op.p.dbg = d;
  rc = launch(op, s, false);
  SF_CHECK_CUDA(cudaMemcpyAsync(stamps, d, 12 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  SF_CHECK_CUDA(cudaStreamSynchronize(s));
  cudaFree(d);
  return rc;
}

// Debug timing: plan once, launch `iters` times back to back between two
// events (F32 epilogue); *us = average device time per launch.
extern "C" int sf_dbg_gemm_time(const void* A, int rows_a, const void* B, int rows_b, int K, int bn,
                                int splits, int swap_ab, void* out, int iters, int pdl, float* us,
                                void* stream) {
  using namespace sf::gemm;
  EpiArgs e{};
  e.kind = EPI_F32;
  e.M = swap_ab ? rows_b : rows_a;
  e.N = swap_ab ? rows_a : rows_b;
  e.out_f32 = static_cast<float*>(out);
  e.ld_f32 = e.N;
  e.inv_width = 1.f;
  e.eps = 1e-6f;
  Op op;
  int rc = plan(&op, A, rows_a, K, B, rows_b, K, K, bn, splits, swap_ab, e);
  DbgWs dws;
  if (!rc) rc = attach_ws(op, dws);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  for (int i = 0; i < 3; ++i)
    if ((rc = launch(op, s, pdl != 0))) return rc;
  cudaEvent_t a, b;
  SF_CHECK_CUDA(cudaEventCreate(&a));
  SF_CHECK_CUDA(cudaEventCreate(&b));
  SF_CHECK_CUDA(cudaEventRecord(a, s));
  for (int i = 0; i < iters; ++i)
    if ((rc = launch(op, s, pdl != 0))) return rc;
  SF_CHECK_CUDA(cudaEventRecord(b, s));
  SF_CHECK_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *us = ms * 1e3f / (float)iters;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return SF_OK;
}
