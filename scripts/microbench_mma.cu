// tcgen05.mma (kind::f16, SS operands, SWIZZLE_128B K-major) issue-to-
// completion time per instruction at small N, on one SM: why the batch-1
// engine's GEMM stages spend ~0.25 us per 4-MMA k-block after the operands
// are resident. Sweeps M, N, the number of independent accumulators and the
// MMA count; prints cycles per MMA (issue) and per MMA (complete).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_13778_b200/csrc -o scripts/mbm scripts/microbench_mma.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace sf;
__device__ int g_random;

// nwarps > 1: warps 0..nwarps-1 each issue n / nwarps MMAs into their own accumulator
// (independent chains), each with its own commit barrier.
__global__ void __launch_bounds__(128, 1) k_mma(int M, int N, int nacc, int n, int reps, long long* out, int nwarps,
                                                int predesc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* A = base;              // 4 k-blocks x 128 rows x 128 B
  uint8_t* B = base + 65536;      // 4 k-blocks x 256 rows x 128 B
  __shared__ __align__(8) uint64_t done_w[4];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (65536 + 131072) / 16; i += blockDim.x) {
    if (g_random) {
      // random bf16 in [-2, 2): sign, exponent 126..128, random mantissa
      uint32_t v[4];
      for (int k = 0; k < 4; ++k) {
        uint32_t h = (uint32_t)(i * 4 + k) * 2654435761u;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        const uint32_t lo = ((h & 0x8000u) | ((126u + (h >> 16) % 3u) << 7) | ((h >> 4) & 0x7Fu));
        const uint32_t hi = (((h >> 1) & 0x8000u) | ((126u + (h >> 20) % 3u) << 7) | ((h >> 9) & 0x7Fu));
        v[k] = lo | (hi << 16);
      }
      reinterpret_cast<uint4*>(base)[i] = make_uint4(v[0], v[1], v[2], v[3]);
    } else {
      reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3f803f80u, 0, 0x3f80u, 0);
    }
  }
  if (threadIdx.x == 0) {
    for (int w = 0; w < 4; ++w) sm100::mbar_init(&done_w[w], 1);
    sm100::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) sm100::tmem_alloc<512>(&tslot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < nwarps) {
    uint64_t* done = &done_w[w];
    const uint32_t idesc = sm100::make_idesc_bf16(M, N);
    const uint32_t a0 = sm100::smem_u32(A), b0 = sm100::smem_u32(B);
    const int acc_cols = N, nw = n / nwarps;
    const uint64_t da0 = sm100::make_sw128_desc(a0), db0 = sm100::make_sw128_desc(b0);
    long long issue = 0, total = 0;
    for (int r = 0; r < reps; ++r) {
      const long long t0 = clock64();
      if (predesc) {
        for (int i = 0; i < nw; ++i) {
          const int kb = (i >> 2) & 3, kk = i & 3;
          sm100::umma_bf16(tmem + (w * nacc + (i >> 2) % nacc) * acc_cols, da0 + (uint64_t)(kb * 1024 + kk * 2),
                           db0 + (uint64_t)(kb * 2048 + kk * 2), idesc, i >= 4 * nacc ? 1u : (kk != 0));
          if (predesc >= 2 && (i & 3) == 3) sm100::umma_commit(&done_w[3]);  // a commit every 4 MMAs
          if (predesc >= 3 && (i & 3) == 3) sm100::tc_fence_after();
        }
      } else {
        for (int i = 0; i < nw; ++i) {
          const int kb = (i >> 2) & 3, kk = i & 3;
          const int a = w * nacc + (i >> 2) % nacc;
          sm100::umma_bf16(tmem + a * acc_cols, sm100::make_sw128_desc(a0 + kb * 16384 + kk * 32),
                           sm100::make_sw128_desc(b0 + kb * 32768 + kk * 32), idesc, i >= 4 * nacc ? 1u : (kk != 0));
        }
      }
      const long long t1 = clock64();
      sm100::umma_commit(done);
      sm100::mbar_wait(done, r & 1);
      const long long t2 = clock64();
      if (r > 0) issue += t1 - t0, total += t2 - t0;
    }
    out[2 * w] = issue / (reps - 1);
    out[2 * w + 1] = total / (reps - 1);
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (threadIdx.x < 32) sm100::tmem_dealloc<512>(tmem);
}

int main() {
  long long* out;
  cudaMalloc(&out, 64);
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct V {
    int M, N, nacc, n, nwarps, predesc;
  } vs[] = {{64, 64, 1, 64, 1, 0},   {128, 64, 1, 64, 1, 0},  {128, 64, 1, 16, 1, 0},  {128, 128, 1, 64, 1, 0},
            {128, 256, 1, 64, 1, 0}, {128, 208, 1, 64, 1, 0}, {64, 64, 1, 4, 1, 0},    {64, 64, 1, 64, 1, 1},
            {128, 64, 1, 64, 1, 1},  {128, 64, 1, 64, 2, 1},  {128, 64, 1, 64, 4, 1},  {64, 64, 1, 64, 4, 1},
            {128, 64, 1, 64, 2, 0},  {128, 64, 1, 64, 4, 0},  {128, 208, 1, 64, 1, 1}, {128, 128, 1, 64, 1, 1},
            {64, 64, 1, 64, 1, 2},   {128, 64, 1, 64, 1, 2},  {64, 64, 1, 64, 1, 3},   {128, 208, 1, 64, 1, 2},
            {64, 64, 1, 64, 2, 2},   {128, 64, 1, 64, 2, 2},  {128, 56, 1, 64, 1, 1},  {64, 56, 1, 64, 1, 1},
            {64, 56, 1, 63, 3, 1},   {128, 56, 1, 63, 3, 1},  {64, 64, 1, 63, 3, 1}};
  for (int rnd = 1; rnd < 2; ++rnd) {
  cudaMemcpyToSymbol(g_random, &rnd, sizeof(int));
  printf("operands: %s\n", rnd ? "random bf16" : "constant pattern");
  for (const V& v : vs) {
    k_mma<<<1, 128, 200 * 1024>>>(v.M, v.N, v.nacc, v.n, 20, out, v.nwarps, v.predesc);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[8] = {0};
    cudaMemcpy(h, out, 16 * v.nwarps, cudaMemcpyDeviceToHost);
    for (int w = 1; w < v.nwarps; ++w) h[0] = h[0] > h[2 * w] ? h[0] : h[2 * w], h[1] = h[1] > h[2 * w + 1] ? h[1] : h[2 * w + 1];
    printf("warps=%d predesc=%d ", v.nwarps, v.predesc);
    printf("M=%3d N=%3d acc=%d n=%3d: issue %6lld cyc (%5.1f/MMA)  complete %6lld cyc (%6.1f/MMA)  floor %5.1f [%s]\n",
           v.M, v.N, v.nacc, v.n, h[0], (double)h[0] / v.n, h[1], (double)h[1] / v.n,
           (v.M > 128 ? v.M : 128) * v.N / 256.0, cudaGetErrorString(e));
  }
  }
  return 0;
}
