// DSMEM exchange microbenchmark (sm_100a): an all-to-all of per-CTA slices
// inside a thread-block cluster (the split-K / split-KV reduction pattern).
// Each of C CTAs owns `bytes` of staged partials in SMEM; slice j goes to
// cluster rank j. Variants: (push) cp.async.bulk shared::cta ->
// shared::cluster with complete_tx on the receiver's mbarrier; (pull)
// 256 threads ld.shared::cluster.v4 of the peers' slices.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbds scripts/microbench_dsmem.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}

__global__ void xchg(int bytes, int mode, unsigned long long* out_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), me = cl.block_rank();
  uint8_t* src = smem;           // [C][slice]
  uint8_t* rx = smem + bytes;    // [C][slice]
  const int slice = bytes / C;
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) reinterpret_cast<float*>(src)[i] = 1.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes)
                 : "memory");
  }
  cl.sync();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (mode == 0) {
    if (threadIdx.x < C) {
      const int j = threadIdx.x;
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              mapa(su32(rx + me * slice), j)),
          "r"(su32(src + j * slice)), "r"(slice), "r"(mapa(su32(&bar), j))
          : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n\t}"
          : "=r"(done)
          : "r"(su32(&bar))
          : "memory");
  } else {
    // pull: rx[j] = peer j's src slice `me`
    float acc = 0.f;
    const int n4 = slice / 16;
    for (int j = 0; j < C; ++j) {
      const uint32_t base = mapa(su32(src + me * slice), j);
      for (int i = threadIdx.x; i < n4; i += blockDim.x * 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * blockDim.x < n4)
            asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                         : "r"(base + (i + u * blockDim.x) * 16));
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * blockDim.x < n4) acc += v[u].x + v[u].y + v[u].z + v[u].w;
      }
    }
    if (acc == 12345.f) out_ns[255] = 1;
  }
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) out_ns[blockIdx.x] = t1 - t0;
  cl.sync();
}

int main() {
  unsigned long long* ns;
  cudaMalloc(&ns, 256 * sizeof(unsigned long long));
  unsigned long long h[256];
  cudaFuncSetAttribute(xchg, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(xchg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 2; ++mode)
    for (int C : {2, 4, 8, 16})
      for (int kb : {32, 64, 104}) {
        const int bytes = kb * 1024;
        cudaLaunchConfig_t cfg{};
        const int grid = (128 / C) * C;
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = 2 * bytes;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = C;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        for (int rep = 0; rep < 3; ++rep) cudaLaunchKernelEx(&cfg, xchg, bytes, mode, ns);
        cudaDeviceSynchronize();
        cudaMemcpy(h, ns, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double avg = 0, mx = 0;
        for (int i = 0; i < grid; ++i) {
          avg += h[i];
          mx = h[i] > mx ? h[i] : mx;
        }
        avg /= grid;
        printf("%s C=%2d %3d KB per CTA: avg %.2f us max %.2f us -> %.1f GB/s per CTA in  [%s]\n",
               mode ? "pull" : "push", C, kb, avg * 1e-3, mx * 1e-3, bytes / avg,
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
