// Ingress microbenchmark for the batch-1 engine's activation loads: why does
// a CTA receive an 8 KB k-block only every ~0.29 us after the grid barrier?
// Pattern (b1engine.cuh): every CTA writes its slice of a 128 KB activation
// image with st.global.cg, grid barrier, then `consumers` CTAs bulk-load the
// whole image as 16 k-blocks of 8 KB through an 11-slot ring (slot reuse
// waits for the previous copy into it to land). Variants isolate the source
// state, the copy size, the L2 cache hint and the consumer count.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbi scripts/microbench_ingress.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncthreads();
}
__device__ int g_wait_mode;  // 0 try_wait, 1 test_wait spin, 2 try_wait with a 20 ns suspend hint
__device__ __forceinline__ bool try_wait(uint32_t a, uint32_t ph) {
  uint32_t done;
  if (g_wait_mode == 1)
    asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(a), "r"(ph)
                 : "memory");
  else if (g_wait_mode == 2)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(ph), "r"(20)
        : "memory");
  else
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(a), "r"(ph)
                 : "memory");
  return done;
}

// flags: 1 = write the image in-kernel before each rep (else read-only, L2-hot)
//        2 = evict_last cache hint on the loads
//        4 = also stream `hbm` (large buffer) on the non-consumer CTAs
struct Args {
  uint8_t* img;       // 128 KB
  const uint8_t* hbm; // large buffer for background streaming
  size_t hbm_bytes;
  unsigned* bar;
  unsigned long long* out;  // [reps][grid][3]: t(barrier pass), t(first block), t(last block)
  int piece, slots, consumers, reps, flags;
};

__global__ void __launch_bounds__(128, 1) k_ingress(Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16];
  const int c = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 16; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const int total = 131072, npieces = total / a.piece;
  uint32_t phase = 0;  // bit per slot
  unsigned epoch = 0;
  for (int r = 0; r < a.reps; ++r) {
    if (a.flags & 1) {
      // every CTA writes 128 KB / grid of the image (16 B units, .cg)
      const int units = total / 16;
      for (int u = c * blockDim.x + threadIdx.x; u < units; u += gridDim.x * blockDim.x)
        __stcg(reinterpret_cast<uint4*>(a.img) + u, make_uint4(u, r, c, 7));
    }
    grid_sync(a.bar, ++epoch * gridDim.x);
    unsigned long long t0 = gtime(), t1 = 0, t2 = 0;
    if (c < a.consumers && (a.flags & 32)) {
      if (threadIdx.x == 0) {
        const int per = npieces / a.slots;
        for (int b = 0; b < a.slots; ++b)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[b])),
                       "r"(per * a.piece)
                       : "memory");
        for (int k = 0; k < npieces; ++k)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(smem + k * a.piece)),
              "l"(a.img + (size_t)k * a.piece), "r"(a.piece), "r"(su32(&full[k / per]))
              : "memory");
        for (int b = 0; b < a.slots; ++b) {
          while (!try_wait(su32(&full[b]), (phase >> b) & 1)) {
          }
          phase ^= 1u << b;
          if (b == 0) t1 = gtime();
        }
        t2 = gtime();
      }
    } else if (c < a.consumers && (a.flags & 16)) {
      if (threadIdx.x == 0) {
        const uint32_t fb = su32(&full[0]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(total) : "memory");
        for (int k = 0; k < npieces; ++k)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(smem + k * a.piece)),
              "l"(a.img + (size_t)k * a.piece), "r"(a.piece), "r"(fb)
              : "memory");
        while (!try_wait(fb, phase & 1)) {
        }
        phase ^= 1u;
        t1 = t2 = gtime();
      }
    } else if (c < a.consumers && (a.flags & 8)) {
      if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        if (l < npieces) {
          const uint32_t fb = su32(&full[l]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(a.piece) : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(smem + l * a.piece)),
              "l"(a.img + (size_t)l * a.piece), "r"(a.piece), "r"(fb)
              : "memory");
        }
        __syncwarp();
        if (l == 0) {
          for (int k = 0; k < npieces; ++k) {
            while (!try_wait(su32(&full[k]), (phase >> k) & 1)) {
            }
            phase ^= 1u << k;
            if (k == 0) t1 = gtime();
          }
          t2 = gtime();
        }
      }
    } else if (c < a.consumers) {
      if (threadIdx.x == 0) {
        int issued = 0, landed = 0;
        while (landed < npieces) {
          while (issued < npieces && issued - landed < a.slots) {
            const int s = issued % a.slots;
            const uint32_t fb = su32(&full[s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(a.piece) : "memory");
            if (a.flags & 2)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
                  "[%3], %4;" ::"r"(su32(smem + s * a.piece)),
                  "l"(a.img + (size_t)issued * a.piece), "r"(a.piece), "r"(fb), "l"(pol)
                  : "memory");
            else
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      su32(smem + s * a.piece)),
                  "l"(a.img + (size_t)issued * a.piece), "r"(a.piece), "r"(fb)
                  : "memory");
            ++issued;
          }
          const int s = landed % a.slots;
          while (!try_wait(su32(&full[s]), (phase >> s) & 1)) {
          }
          phase ^= 1u << s;
          if (landed == 0) t1 = gtime();
          ++landed;
        }
        t2 = gtime();
      }
    } else if (a.flags & 4) {
      // background HBM stream: 32 KB bulk copies, 4 in flight, ~1 MB per CTA
      if (threadIdx.x == 0) {
        const size_t per = (a.hbm_bytes / gridDim.x) & ~(size_t)32767;
        const uint8_t* src = a.hbm + per * c + (size_t)r * 0;
        int issued = 0, landed = 0;
        const int n = (int)(per / 32768) < 32 ? (int)(per / 32768) : 32;
        while (landed < n) {
          while (issued < n && issued - landed < 4) {
            const int s = issued % 4;
            const uint32_t fb = su32(&full[s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(32768) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(smem + s * 32768)),
                "l"(src + (size_t)issued * 32768), "r"(32768), "r"(fb)
                : "memory");
            ++issued;
          }
          const int s = landed % 4;
          while (!try_wait(su32(&full[s]), (phase >> s) & 1)) {
          }
          phase ^= 1u << s;
          ++landed;
        }
      }
    }
    if (threadIdx.x == 0) {
      unsigned long long* o = a.out + ((size_t)r * gridDim.x + c) * 3;
      o[0] = t0, o[1] = t1, o[2] = t2;
    }
    grid_sync(a.bar, ++epoch * gridDim.x);
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm, reps = 20;
  uint8_t *img, *hbm;
  unsigned* bar;
  unsigned long long* out;
  const size_t hbm_bytes = (size_t)1 << 30;
  cudaMalloc(&img, 131072);
  cudaMalloc(&hbm, hbm_bytes);
  cudaMemset(hbm, 1, hbm_bytes);
  cudaMemset(img, 0, 131072);
  cudaMalloc(&bar, 64);
  cudaMalloc(&out, sizeof(unsigned long long) * reps * grid * 3);
  cudaFuncSetAttribute(k_ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  unsigned long long* h = new unsigned long long[reps * grid * 3];
  struct V {
    int piece, slots, consumers, flags;
    const char* name;
  } vs[] = {
      {8192, 11, 40, 1, "written in-kernel, 8 KB x 11 slots, 40 consumers"},
      {8192, 11, 40, 0, "read-only (L2-hot), 8 KB x 11 slots, 40 consumers"},
      {8192, 11, 40, 3, "written, evict_last hint, 8 KB x 11, 40 consumers"},
      {8192, 11, 40, 5, "written + HBM stream on the others, 8 KB x 11, 40 consumers"},
      {8192, 11, 1, 1, "written, 8 KB x 11, 1 consumer"},
      {8192, 11, 128, 1, "written, 8 KB x 11, 128 consumers"},
      {16384, 5, 40, 1, "written, 16 KB x 5 slots, 40 consumers"},
      {32768, 3, 40, 1, "written, 32 KB x 3 slots, 40 consumers"},
      {8192, 2, 40, 1, "written, 8 KB x 2 slots, 40 consumers"},
      {8192, 16, 40, 1, "written, 8 KB x 16 slots, 40 consumers"},
      {65536, 2, 40, 1, "written, 64 KB x 2 slots, 40 consumers"},
      {131072, 1, 40, 1, "written, 128 KB x 1 slot, 40 consumers"},
      {8192, 16, 40, 9, "written, 8 KB x 16, issued by 16 lanes at once"},
      {8192, 16, 40, 17, "written, 8 KB x 16 on ONE mbarrier (one thread)"},
      {16384, 8, 40, 17, "written, 16 KB x 8 on ONE mbarrier (one thread)"},
      {2048, 64, 40, 17, "written, 2 KB x 64 on ONE mbarrier (one thread)"},
      {8192, 2, 40, 33, "written, 8 KB x 16 all in flight, 2 mbarriers"},
      {8192, 4, 40, 33, "written, 8 KB x 16 all in flight, 4 mbarriers"},
      {8192, 8, 40, 33, "written, 8 KB x 16 all in flight, 8 mbarriers"},
      {8192, 16, 40, 33, "written, 8 KB x 16 all in flight, 16 mbarriers"},
      {32768, 4, 40, 33, "written, 32 KB x 4 all in flight, 4 mbarriers"},
  };
  for (int mode = 0; mode < 1; ++mode) {
  cudaMemcpyToSymbol(g_wait_mode, &mode, sizeof(int));
  printf("wait mode %d (%s)\n", mode, mode == 0 ? "try_wait" : mode == 1 ? "test_wait spin" : "try_wait, 20 ns hint");
  for (const V& v : vs) {
    Args a{img, hbm, hbm_bytes, bar, out, v.piece, v.slots, v.consumers, reps, v.flags};
    cudaMemset(bar, 0, 64);
    void* args[] = {&a};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_ingress, grid, 128, args, 200 * 1024, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, sizeof(unsigned long long) * reps * grid * 3, cudaMemcpyDeviceToHost);
    // per rep: median over consumers of (first - t0, last - t0) relative to that consumer's barrier pass
    double first = 0, last = 0;
    int n = 0;
    for (int r = 2; r < reps; ++r)
      for (int c = 0; c < v.consumers; ++c) {
        const unsigned long long* o = h + ((size_t)r * grid + c) * 3;
        first += (double)(o[1] - o[0]);
        last += (double)(o[2] - o[0]);
        ++n;
      }
    first /= n, last /= n;
    printf("%-62s first %6.2f us  all 128 KB %6.2f us  -> %6.1f GB/s per SM [%s]\n", v.name, first * 1e-3,
           last * 1e-3, 131072.0 / last, cudaGetErrorString(e));
  }
  }
  return 0;
}
