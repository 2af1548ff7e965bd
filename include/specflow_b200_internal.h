/*
 * specflow_b200 internal kernel entry points — unit-test hooks for the
 * pi0-scale building blocks (not part of the reference-facing boundary).
 * Same conventions as specflow_b200.h.
 */
#ifndef SPECFLOW_B200_INTERNAL_H
#define SPECFLOW_B200_INTERNAL_H

#include <stddef.h>

#include "specflow_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* D[m, n] = sum_k A[m|n, k] B[n|m, k] through the tcgen05 GEMM (bf16 in, fp32
 * accumulate). swap_ab=0: A rows are output rows m, B rows are features n;
 * swap_ab=1: A rows are features n, B rows are output rows m. epi_kind 0 stores
 * fp32, 1 stores bf16; if `ssq` is non-NULL each output row m is scaled by
 * rsqrt(sum_g ssq[g*ssq_ld + m] * inv_width + 1e-6) (RMSNorm folded into the
 * epilogue). splits <= 0 picks split-K automatically. Synchronises `stream`. */
int sf_dbg_gemm(const void* A, int rows_a, const void* B, int rows_b, int K, int bn, int splits,
                int swap_ab, int epi_kind, void* out, int ld_out, int M_valid, int N_valid,
                const float* ssq, int ssq_groups, int ssq_ld, float inv_width, void* stream);

/* %globaltimer stamps (ns, 12 entries) of block (0,0,0) of one warm launch of
 * a swap-AB split-K GEMM (see gemm.cu for the stamp points). */
int sf_dbg_gemm_trace(const void* A, int rows_a, const void* B, int rows_b, int K, int bn,
                      int splits, void* out, unsigned long long* stamps, void* stream);

/* Average device time (us) of `iters` back-to-back launches of one planned
 * GEMM (fp32 store epilogue), optionally with programmatic dependent launch. */
int sf_dbg_gemm_time(const void* A, int rows_a, const void* B, int rows_b, int K, int bn,
                     int splits, int swap_ab, void* out, int iters, int pdl, float* us,
                     void* stream);

/* Per-stage %globaltimer stamps of the last batch-1 engine launch run with
 * SF_B1_TRACE set: [148 CTAs][stages][4] (stage start, operand ready,
 * accumulator / softmax done, stage done), copied to host `out` (n entries). */
int sf_ae_b1_trace(void* ae_handle, unsigned long long* out, size_t n);

/* %globaltimer stamps of the fused tiny flash round (cluster rank 0): on != 0
 * enables them for the following launches; `out` (32 entries, may be NULL)
 * receives the stamps of the last launch (0 start, 1 weights issued, 8-15
 * draft layers done, 2 branches packed, 16-23 field layers done, 3 end). */
int sf_tiny_trace(int on, unsigned long long* out);

#ifdef __cplusplus
}
#endif

#endif
