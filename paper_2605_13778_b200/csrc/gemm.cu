// Host side of the tcgen05 GEMM: tensor maps, split-K planning, PDL launch,
// and a debug C entry point used by the GEMM unit tests.

#include <cudaTypedefs.h>
#include <stdio.h>

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

size_t ws_bytes_needed(int rows_a, int rows_b, int K, int bn, int splits) {
  const int tiles = ((rows_a + BM - 1) / BM) * ((rows_b + bn - 1) / bn);
  (void)K;
  return splits > 1 ? (size_t)splits * tiles * bn * BM * sizeof(float) : 0;
}

int plan(Op* op, const void* A, int rows_a, int lda, const void* B, int rows_b, int ldb, int K,
         int bn, int splits, int swap_ab, const EpiArgs& e, float* ws, size_t ws_bytes,
         int* counters, int n_counters, int max_stages) {
  SF_REQUIRE(bn >= 16 && bn <= 256 && bn % 16 == 0, "bn must be a multiple of 16 in [16, 256]");
  SF_REQUIRE(K % BK == 0, "K (%d) must be a multiple of %d", K, BK);
  SF_REQUIRE(e.kind != EPI_RESID || swap_ab || bn % 128 == 0, "residual epilogue needs bn %% 128 == 0");
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
  const int tiles = p.tiles_a * p.tiles_b;
  if (splits <= 0) {
    // cover the 148 SMs with weight streams: split K until tiles*splits >= ~148
    splits = (148 + tiles - 1) / tiles;
  }
  splits = splits < 1 ? 1 : (splits > p.num_kb ? p.num_kb : splits);
  p.kb_per_split = (p.num_kb + splits - 1) / splits;
  p.splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;  // every split gets >= 1 block
  if (p.splits > 1) {
    SF_REQUIRE(ws && counters, "split-K needs a workspace");
    SF_REQUIRE(ws_bytes >= ws_bytes_needed(rows_a, rows_b, K, bn, p.splits),
               "split-K workspace too small");
    SF_REQUIRE(n_counters >= tiles, "split-K counters too small");
  }
  p.ws = ws;
  p.counters = counters;
  p.e = e;
  const uint32_t stage_bytes = kAStageBytes + ((bn * BK * 2 + 1023) & ~1023);
  const size_t scratch = 64 + 256 * 4 + 4 * 256 * 4 + 1024 /* align slack */;
  int stages = (int)((227 * 1024 - scratch) / stage_bytes);
  if (stages > max_stages) stages = max_stages;
  if (stages > p.kb_per_split) stages = p.kb_per_split < 2 ? 2 : p.kb_per_split;
  SF_REQUIRE(stages >= 2, "GEMM tile does not fit in shared memory");
  p.stages = stages;
  op->smem = (size_t)stages * stage_bytes + 8 * (2 * stages + 1) + 16 + 256 * 4 + 4 * 256 * 4 + 1024;
  op->grid = dim3(p.tiles_a, p.tiles_b, p.splits);
  int rc = make_map(&op->ta, A, rows_a, K, lda, BM);
  if (rc) return rc;
  return make_map(&op->tb, B, rows_b, K, ldb, bn);
}

int launch(const Op& op, cudaStream_t stream, bool pdl) {
  static bool attr_set = false;
  if (!attr_set) {
    SF_CHECK_CUDA(cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = op.grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = op.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, gemm_kernel, op.ta, op.tb, op.p));
  count_launch();
  return SF_OK;
}

}  // namespace gemm
}  // namespace sf

// Debug entry: D = A @ B^T with an F32 / BF16 epilogue (optional RMS row
// scale from ssq partials). Allocates its own split-K workspace; not for the
// hot path.
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
  const int tiles = ((rows_a + BM - 1) / BM) * ((rows_b + bn - 1) / bn);
  const int max_splits = K / BK;
  const size_t wsb = ws_bytes_needed(rows_a, rows_b, K, bn, splits > 0 ? splits : max_splits);
  float* ws = nullptr;
  int* counters = nullptr;
  if (wsb) SF_CHECK_CUDA(cudaMalloc(&ws, wsb));
  SF_CHECK_CUDA(cudaMalloc(&counters, sizeof(int) * (tiles + 1)));
  SF_CHECK_CUDA(cudaMemsetAsync(counters, 0, sizeof(int) * (tiles + 1), (cudaStream_t)stream));
  Op op;
  int rc = plan(&op, A, rows_a, K, B, rows_b, K, K, bn, splits, swap_ab, e, ws, wsb, counters,
                tiles + 1);
  if (!rc) rc = launch(op, (cudaStream_t)stream, false);
  cudaStreamSynchronize((cudaStream_t)stream);
  if (ws) cudaFree(ws);
  cudaFree(counters);
  return rc;
}
