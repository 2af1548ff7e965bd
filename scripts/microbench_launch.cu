// Launch-overhead microbenchmark on sm_100a: back-to-back device time per
// launch for empty / clustered / big-SMEM / TMEM-allocating kernels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_launch.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void k_empty() {}

__global__ void k_cluster_sync() {
  cg::this_cluster().sync();
}

__global__ void k_smem(int n) {
  extern __shared__ float s[];
  if (threadIdx.x < n) s[threadIdx.x] = 0.f;
}

__global__ void k_tmem() {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot));
}

template <typename F>
float time_it(F launch, int iters = 2000) {
  for (int i = 0; i < 20; ++i) launch();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / iters;
}

void cluster_launch(void (*k)(), int grid, int cluster, int threads, size_t smem) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k);
}

int main() {
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_cluster_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("empty 1x32            : %6.2f us\n", time_it([] { k_empty<<<1, 32>>>(); }));
  printf("empty 148x320         : %6.2f us\n", time_it([] { k_empty<<<148, 320>>>(); }));
  printf("smem 200KB 148x320    : %6.2f us\n",
         time_it([] { k_smem<<<148, 320, 200 * 1024>>>(320); }));
  printf("smem 100KB 148x320    : %6.2f us\n",
         time_it([] { k_smem<<<148, 320, 100 * 1024>>>(320); }));
  printf("tmem alloc 148x320    : %6.2f us\n", time_it([] { k_tmem<<<148, 320>>>(); }));
  for (int c : {1, 2, 8, 16}) {
    const int grid = c == 1 ? 128 : 128;
    printf("cluster.sync c=%2d g=%d: %6.2f us\n", c, grid,
           time_it([&] { cluster_launch(k_cluster_sync, grid, c, 256, 0); }));
  }
  printf("cluster.sync c=16 g=16: %6.2f us\n",
         time_it([&] { cluster_launch(k_cluster_sync, 16, 16, 256, 0); }));
  printf("cluster.sync c=8 g=8  : %6.2f us\n",
         time_it([&] { cluster_launch(k_cluster_sync, 8, 8, 256, 0); }));
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
