// L2 -> SMEM ingress microbenchmark (sm_100a): per-CTA bulk-copy
// (cp.async.bulk) throughput from an L2-resident buffer, by CTA count and
// ring depth. One elected thread streams `chunks` 16 KB chunks through a
// `stages`-deep mbarrier ring; the same thread consumes (waits) them.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbl2 scripts/microbench_l2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ingest(const uint8_t* src, size_t src_bytes, int chunks, int stages, int chunk_bytes,
                       unsigned long long* out_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[32];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  size_t off = ((size_t)blockIdx.x * (src_bytes / gridDim.x / chunk_bytes) * chunk_bytes) % src_bytes;
  auto issue = [&](int i) {
    const int s = i % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])),
                 "r"(chunk_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(smem + (size_t)s * chunk_bytes)),
        "l"(src + off), "r"(chunk_bytes), "r"(su32(&bars[s]))
        : "memory");
    off += chunk_bytes;
    if (off + chunk_bytes > src_bytes) off = 0;
  };
  for (int i = 0; i < stages && i < chunks; ++i) issue(i);
  for (int i = 0; i < chunks; ++i) {
    const int s = i % stages;
    const uint32_t par = (i / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
          : "=r"(done)
          : "r"(su32(&bars[s])), "r"(par)
          : "memory");
    if (i + stages < chunks) issue(i + stages);
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out_ns[blockIdx.x] = t1 - t0;
}

int main() {
  for (size_t bytes : {48ull << 20, 4096ull << 20}) {  // L2-resident, then HBM-streaming
  printf("source %zu MB\n", bytes >> 20);
  uint8_t* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  unsigned long long* ns;
  cudaMalloc(&ns, 256 * sizeof(unsigned long long));
  unsigned long long h[256];
  cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int chunk = 16384;
  for (int ctas : {1, 16, 64, 128, 148}) {
    for (int stages : {2, 4, 8, 12}) {
      const int chunks = 256;  // 4 MB per CTA
      for (int rep = 0; rep < 2; ++rep)
        ingest<<<ctas, 32, stages * chunk>>>(src, bytes, chunks, stages, chunk, ns);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      ingest<<<ctas, 32, stages * chunk>>>(src, bytes, chunks, stages, chunk, ns);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(h, ns, ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      double avg = 0;
      for (int i = 0; i < ctas; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        avg += h[i];
      }
      avg /= ctas;
      const double per_cta = (double)chunks * chunk;
      printf("ctas=%3d stages=%2d: per-CTA %.1f GB/s (avg ns %.0f), chip %.2f TB/s (event %.3f ms)\n",
             ctas, stages, per_cta / avg, avg, per_cta * ctas / (mx * 1e-9) / 1e12, ms);
    }
  }
  cudaFree(src);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
