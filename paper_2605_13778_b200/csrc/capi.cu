// C-ABI plumbing: thread-local error message, version, launch counter.
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "common.cuh"

namespace sf {
namespace {
thread_local char g_err[1024] = {0};
std::atomic<int64_t> g_launches{0};
}  // namespace

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace sf

extern "C" const char* sf_last_error(void) { return sf::g_err; }

extern "C" int sf_version(void) { return 1; }

extern "C" int64_t sf_launch_count(int reset) {
  if (reset) return sf::g_launches.exchange(0);
  return sf::g_launches.load();
}

// Host <-> device staging of one round's packed inputs / outputs (pinned host
// buffers): one ctypes call each instead of torch copy_ + stream lookup +
// synchronize (~3x less host time per tiny round).
extern "C" int sf_copy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  SF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return SF_OK;
}

extern "C" int sf_copy_d2h_sync(void* dst, const void* src, size_t bytes, void* stream) {
  SF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  SF_CHECK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return SF_OK;
}
