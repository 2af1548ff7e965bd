// Batch-1 dataflow primitives on sm_100a, all 148 SMs concurrently (one CTA
// per SM, 256 threads), device-timed with CUDA events over many repetitions:
//   egress   : per-CTA fp32 tile (32 KB / 106 KB) written / reduced into L2:
//              st.global.v4, st.global.v8, red.global.add.v4.f32,
//              cp.reduce.async.bulk .add.f32 (SMEM source), cp.async.bulk store
//   ingress  : per-CTA bulk copy L2 -> SMEM (cp.async.bulk, mbarrier)
//   barrier  : grid-wide barrier (release-add + acquire spin) round trip
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbp scripts/microbench_b1prims.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__global__ void k_barrier(unsigned* bar, int reps) {
  for (int r = 1; r <= reps; ++r) grid_sync(bar, r * gridDim.x);
}

// mode: 0 st.v4, 1 st.v8, 2 red.add.v4.f32, 3 bulk reduce add.f32, 4 bulk store
// dst per CTA: contiguous `bytes`; `shared` != 0 -> all CTAs of a group of 8
// target the same region (real split-K reduction contention).
__global__ void k_egress(float* ws, int bytes, int mode, int reps, int shared) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int n4 = bytes / 16;
  const size_t region = shared ? (size_t)(blockIdx.x / 8) : (size_t)blockIdx.x;
  float* mine = ws + region * (bytes / 4);
  if (mode >= 3) {
    for (int i = threadIdx.x; i < n4; i += blockDim.x)
      reinterpret_cast<float4*>(smem)[i] = make_float4(1.f, 2.f, 3.f, 4.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    if (mode == 0) {
      for (int i = threadIdx.x; i < n4; i += blockDim.x)
        __stcg(reinterpret_cast<float4*>(mine) + i, make_float4(1.f, 2.f, 3.f, (float)i));
    } else if (mode == 1) {
      for (int i = threadIdx.x; i < n4 / 2; i += blockDim.x) {
        float* p = mine + 8 * i;
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(1.f), "f"(2.f),
                     "f"(3.f), "f"(4.f), "f"(5.f), "f"(6.f), "f"(7.f), "f"((float)i)
                     : "memory");
      }
    } else if (mode == 2) {
      for (int i = threadIdx.x; i < n4; i += blockDim.x) {
        float* p = mine + 4 * i;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(2.f), "f"(3.f),
                     "f"(4.f)
                     : "memory");
      }
    } else {
      if (threadIdx.x == 0) {
        const int chunk = 16384;
        for (int off = 0; off < bytes; off += chunk) {
          const int sz = bytes - off < chunk ? bytes - off : chunk;
          if (mode == 3)
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                             reinterpret_cast<uint8_t*>(mine) + off),
                         "r"(su32(smem + off)), "r"(sz)
                         : "memory");
          else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                             reinterpret_cast<uint8_t*>(mine) + off),
                         "r"(su32(smem + off)), "r"(sz)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
    }
    __syncthreads();
  }
}

// per-CTA bulk copy L2 -> SMEM of `bytes` (in 16 KB pieces), reps times
__global__ void k_ingress(const float* src, int bytes, int reps, int same) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar;
  const uint8_t* g = reinterpret_cast<const uint8_t*>(src) + (same ? 0 : (size_t)blockIdx.x * bytes);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar)), "r"(bytes)
                   : "memory");
      for (int off = 0; off < bytes; off += 16384)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(smem + off)),
            "l"(g + off), "r"(16384), "r"(su32(&mbar))
            : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(su32(&mbar)), "r"(r & 1)
            : "memory");
    }
    __syncthreads();
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm;
  float* ws;
  cudaMalloc(&ws, (size_t)grid * 256 * 1024);
  cudaMemset(ws, 0, (size_t)grid * 256 * 1024);
  unsigned* bar;
  cudaMalloc(&bar, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  cudaFuncSetAttribute(k_egress, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("SMs %d\n", nsm);
  for (int reps : {100, 1000}) {
    cudaMemset(bar, 0, 64);
    k_barrier<<<grid, 256>>>(bar, 10);
    cudaMemset(bar, 0, 64);
    cudaEventRecord(e0);
    k_barrier<<<grid, 256>>>(bar, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid barrier x%d: %.3f us per barrier [%s]\n", reps, ms * 1e3 / reps,
           cudaGetErrorString(cudaGetLastError()));
  }
  const char* names[] = {"st.v4", "st.v8", "red.add.v4.f32", "bulk reduce add.f32", "bulk store"};
  for (int bytes : {32768, 106496})
    for (int shared : {0, 1})
      for (int mode = 0; mode < 5; ++mode) {
        const int reps = 50;
        k_egress<<<grid, 256, mode >= 3 ? bytes : 0>>>(ws, bytes, mode, 2, shared);
        cudaEventRecord(e0);
        k_egress<<<grid, 256, mode >= 3 ? bytes : 0>>>(ws, bytes, mode, reps, shared);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double per = ms * 1e3 / reps;
        printf("egress %6d B %s %-20s: %.3f us per tile, %.1f GB/s per SM, %.2f TB/s total [%s]\n", bytes,
               shared ? "8-way" : "own  ", names[mode], per, bytes / per * 1e-3, bytes * (double)grid / per * 1e-6,
               cudaGetErrorString(cudaGetLastError()));
      }
  for (int bytes : {32768, 131072})
    for (int same : {0, 1}) {
      const int reps = 50;
      k_ingress<<<grid, 256, bytes>>>(ws, bytes, 2, same);
      cudaEventRecord(e0);
      k_ingress<<<grid, 256, bytes>>>(ws, bytes, reps, same);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double per = ms * 1e3 / reps;
      printf("ingress %6d B %s: %.3f us per copy, %.1f GB/s per SM, %.2f TB/s total [%s]\n", bytes,
             same ? "same src" : "own src ", per, bytes / per * 1e-3, bytes * (double)grid / per * 1e-6,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
