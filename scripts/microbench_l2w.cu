// L2 write microbenchmark (sm_100a): per-CTA partial-tile store throughput
// as in the split-K epilogue (106 KB of fp32 per CTA), then a release-add +
// acquire spin on a counter shared by groups of S CTAs (the tile barrier).
// Modes: 0 = st.global.cg float4 from 256 threads, 1 = TMA bulk store
// (cp.async.bulk.global.shared::cta) from SMEM, 2 = mode 0 without fence/barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbl2w scripts/microbench_l2w.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void writer(float4* ws, int bytes, int mode, int S, unsigned* cnt, unsigned long long* ns) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int n4 = bytes / 16;
  float4* mine = ws + (size_t)blockIdx.x * n4;
  for (int i = threadIdx.x; i < n4 && mode == 1; i += blockDim.x)
    reinterpret_cast<float4*>(smem)[i] = make_float4(1.f, 2.f, 3.f, 4.f);
  __syncthreads();
  unsigned long long t0, t1, t2;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (mode == 0 || mode == 2) {
    for (int i = threadIdx.x; i < n4; i += blockDim.x) __stcg(mine + i, make_float4(1.f, 2.f, 3.f, (float)i));
  } else {
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int chunk = 16384;
      for (int off = 0; off < bytes; off += chunk) {
        const int sz = bytes - off < chunk ? bytes - off : chunk;
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
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (mode != 2 && threadIdx.x == 0) {
    unsigned* c = cnt + blockIdx.x / S;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
    unsigned v = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    } while (v < (unsigned)S);
  }
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
  if (threadIdx.x == 0) {
    ns[2 * blockIdx.x] = t1 - t0;
    ns[2 * blockIdx.x + 1] = t2 - t0;
  }
}

int main() {
  const int ctas = 128, bytes = 128 * 208 * 4;
  float4* ws;
  cudaMalloc(&ws, (size_t)ctas * bytes);
  unsigned* cnt;
  cudaMalloc(&cnt, 4096);
  unsigned long long* ns;
  cudaMalloc(&ns, 2 * ctas * 8);
  unsigned long long h[2 * ctas];
  cudaFuncSetAttribute(writer, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode : {2, 0, 1})
    for (int S : {2, 8, 16}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(cnt, 0, 4096);
        writer<<<ctas, 256, mode == 1 ? bytes : 0>>>(ws, bytes, mode, S, cnt, ns);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, ns, sizeof(h), cudaMemcpyDeviceToHost);
      double a1 = 0, a2 = 0, m2 = 0;
      for (int i = 0; i < ctas; ++i) {
        a1 += h[2 * i];
        a2 += h[2 * i + 1];
        m2 = h[2 * i + 1] > m2 ? h[2 * i + 1] : m2;
      }
      printf("mode %d S=%2d: issue %.2f us, +barrier %.2f us (max %.2f) -> %.1f GB/s per CTA [%s]\n", mode, S,
             a1 / ctas * 1e-3, a2 / ctas * 1e-3, m2 * 1e-3, bytes / (a2 / ctas),
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
