// TMA multicast ingress microbenchmark (sm_100a): per-SM SMEM fill rate when
// the C CTAs of a cluster each issue 1/C of the 16 KB chunks with
// .multicast::cluster (every CTA still receives every chunk), vs C = 1.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbmc scripts/microbench_mcast.cu -lcuda
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void mc(const __grid_constant__ CUtensorMap tm, int chunks, int stages, unsigned long long* ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), me = cl.block_rank();
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(C));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) {
    const uint16_t mask = (uint16_t)((1u << C) - 1);
    const int rows = 128 / C;
    auto issue = [&](int i) {
      const int s = i % stages;
      if (i >= stages) {  // every CTA of the cluster released slot s (chunk i - stages consumed)
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                       : "=r"(ok) : "r"(su32(&empty[s])), "r"(((i / stages) & 1) ^ 1) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(16384) : "memory");
      const int y = (blockIdx.x / C * 4096 + i * 128) % 65536 + me * rows;
      if (C == 1)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(buf + s * 16384)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(y), "r"(su32(&full[s])) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;"
                     ::"r"(su32(buf + s * 16384 + me * rows * 128)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(y),
                     "r"(su32(&full[s])), "h"(mask) : "memory");
    };
    for (int i = 0; i < stages && i < chunks; ++i) issue(i);
    for (int i = 0; i < chunks; ++i) {
      const int s = i % stages;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                     : "=r"(ok) : "r"(su32(&full[s])), "r"((i / stages) & 1) : "memory");
      for (int r = 0; r < C; ++r) {  // consumed: release slot s in every CTA of the cluster
        uint32_t a;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(&empty[s])), "r"(r));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
      }
      if (i + stages < chunks) issue(i + stages);
    }
  }
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) ns[blockIdx.x] = t1 - t0;
  cl.sync();
}

int main() {
  const size_t rows = 65536, cols = 64;  // bf16 [65536][64] = 8 MB, L2 resident
  void* src;
  cudaMalloc(&src, rows * cols * 2);
  cudaMemset(src, 1, rows * cols * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  unsigned long long* ns;
  cudaMalloc(&ns, 256 * 8);
  unsigned long long h[256];
  cudaFuncSetAttribute(mc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(mc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C : {1, 2, 4}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t str[1] = {cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)(128 / C)};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int grid = 148 / C * C, chunks = 512, stages = 8;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = stages * 16384 + 1024;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = C;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 3; ++rep) cudaLaunchKernelEx(&cfg, mc, tm, chunks, stages, ns);
    cudaDeviceSynchronize();
    cudaMemcpy(h, ns, grid * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < grid; ++i) avg += h[i];
    avg /= grid;
    printf("cluster %d (%d CTAs): per-SM SMEM fill %.1f GB/s (received), %.1f GB/s issued [%s]\n", C, grid,
           chunks * 16384.0 / avg, chunks * 16384.0 / C / avg, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
