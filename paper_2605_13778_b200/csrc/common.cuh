// Shared device helpers for the specflow_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "specflow_b200.h"

namespace sf {

// ---- error plumbing (capi.cu owns the thread-local message) --------------
void set_error(const char* fmt, ...);
void count_launch(int n = 1);

#define SF_CHECK_CUDA(expr)                                                        \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::sf::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),      \
                      __FILE__, __LINE__);                                         \
      return SF_ECUDA;                                                             \
    }                                                                              \
  } while (0)

#define SF_REQUIRE(cond, ...)         \
  do {                                \
    if (!(cond)) {                    \
      ::sf::set_error(__VA_ARGS__);   \
      return SF_EINVAL;               \
    }                                 \
  } while (0)

#define SF_DISPATCH(prec, FN, ...)                              \
  ((prec) == SF_F32   ? FN<float>(__VA_ARGS__)                  \
   : (prec) == SF_F64 ? FN<double>(__VA_ARGS__)                 \
                      : (::sf::set_error("unknown precision %d", prec), SF_EINVAL))

// ---- exact (non-contracted) scalar ops so element-wise steps round exactly
// like the reference's numpy expressions -----------------------------------
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float tanh_t(float a) { return tanhf(a); }
__device__ __forceinline__ double tanh_t(double a) { return tanh(a); }
__device__ __forceinline__ bool finite_t(float a) { return isfinite(a); }
__device__ __forceinline__ bool finite_t(double a) { return isfinite(a); }

// numpy's pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) for n <= 128,
// which is what np.sum(..., axis=1) runs on each contiguous row: sequential
// below 8 elements, 8 interleaved accumulators otherwise.
template <typename T, typename F>
__device__ __forceinline__ T numpy_pairwise_sum(int n, F&& term) {
  if (n < 8) {
    T res = T(0);
    for (int i = 0; i < n; ++i) res = add_rn(res, term(i));
    return res;
  }
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = term(j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = add_rn(r[j], term(i + j));
  }
  T res = add_rn(add_rn(add_rn(r[0], r[1]), add_rn(r[2], r[3])),
                 add_rn(add_rn(r[4], r[5]), add_rn(r[6], r[7])));
  for (; i < n; ++i) res = add_rn(res, term(i));
  return res;
}

// continuous distance of one step (actions.py:168-181): l2 = sqrt(sum diff^2)
// compared AFTER the sqrt (Appendix A.1), linf = max |diff|.
template <typename T, typename GA, typename GB>
__device__ __forceinline__ T step_distance(int cdims, int metric, GA&& a, GB&& b) {
  if (metric == SF_METRIC_L2) {
    T s = numpy_pairwise_sum<T>(cdims, [&](int c) {
      T d = sub_rn(a(c), b(c));
      return mul_rn(d, d);
    });
    return sqrt_rn(s);
  }
  T m = T(0);
  for (int c = 0; c < cdims; ++c) {
    T d = fabs(sub_rn(a(c), b(c)));
    m = (c == 0 || d > m || d != d) ? d : m;  // np.max propagates NaN
  }
  return m;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

}  // namespace sf
