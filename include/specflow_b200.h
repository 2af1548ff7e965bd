/*
 * specflow_b200 — C-ABI of the B200-native speculative-replanning path.
 *
 * Drop-in boundary for the reference `specflow` package (arXiv 2605.13778
 * desk-scale restatement, /root/reference/pkg/src/specflow). The reference is
 * pure Python with no FFI; each entry point below names the reference
 * function it replaces (file:line). INTEGRATION.md shows the ctypes binding a
 * maintainer would add on the reference side.
 *
 * Conventions
 *  - Plain pointers and sizes only. Every pointer documented "device" is a
 *    CUDA device pointer; `stream` is a cudaStream_t passed as void*.
 *  - All entry points are asynchronous on `stream` unless stated otherwise and
 *    never allocate on the hot path (handles preallocate their workspaces).
 *  - Return value: SF_OK or one of the SF_E* codes; sf_last_error() returns a
 *    thread-local message. The Python layer maps SF_EINVAL -> ValueError,
 *    SF_ENONFINITE -> FloatingPointError, SF_ERUNTIME -> RuntimeError.
 *  - Device-side non-finite detection is reported in the result words
 *    (sf_verify_out_t.result[SF_RES_NONFINITE] / full-round status) and raised
 *    by the host after the round's single synchronisation.
 */
#ifndef SPECFLOW_B200_H
#define SPECFLOW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SF_OK 0
#define SF_EINVAL 1     /* ValueError */
#define SF_ENONFINITE 2 /* FloatingPointError */
#define SF_ERUNTIME 3   /* RuntimeError */
#define SF_ECUDA 4      /* CUDA launch / driver failure */

#define SF_F32 0 /* fp32 arithmetic (north-star "fp32 mode", rtol 1e-5) */
#define SF_F64 1 /* fp64 arithmetic (reference precision) */

#define SF_MAX_LAYERS 8
#define SF_MAX_K 16

#define SF_METRIC_L2 0
#define SF_METRIC_LINF 1

/* decision codes (runtime.py:286-320) */
#define SF_PATH_FLASH_ACCEPTED 0
#define SF_PATH_FLASH_REJECTED 1 /* "flash_rejected_fallback" */
#define SF_PATH_FLASH_PHASE 2    /* "flash_phase_fallback" */
#define SF_PATH_FULL 3           /* "full" (no cache yet, or full-only mode) */
#define SF_PATH_PERIODIC 4       /* "periodic_refresh" (runtime.py:247-253, :263) */

/* result words written by every verify entry point */
#define SF_RES_PREFIX 0    /* min over branches (verifier.py:147) */
#define SF_RES_SWITCH 1    /* gripper switch in draft or any branch (verifier.py:137-142) */
#define SF_RES_PATH 2      /* SF_PATH_* (runtime.py:286-291) */
#define SF_RES_PLANNED 3   /* min(L, R if prefix_cap else H) or R on fallback (runtime.py:310, :319-320) */
#define SF_RES_NONFINITE 4 /* first branch index with non-finite v/recon, else -1 */
#define SF_RESULT_WORDS 8

/* Tanh MLP (nets.py:16-44): weights (n_out, n_in) row-major with row stride
 * ld[l] >= n_in elements (0 means n_in; a 16-byte multiple lets the kernels
 * stage the layer into shared memory with TMA bulk copies), biases (n_out). */
typedef struct {
  int n_layers;
  int sizes[SF_MAX_LAYERS + 1];
  int ld[SF_MAX_LAYERS];
  const void* w[SF_MAX_LAYERS]; /* device */
  const void* b[SF_MAX_LAYERS]; /* device */
} sf_mlp_t;

/* VerifierConfig (verifier.py:29-50) + the runtime fallback knobs
 * (runtime.py:67-88) the device decision needs. */
typedef struct {
  int k;
  double taus[SF_MAX_K];
  double delta;
  int metric;           /* SF_METRIC_* */
  int window;           /* gripper_window; < 0 scans the full chunk */
  double current_sign;  /* -1.0 or +1.0 (runtime.py:60-64) */
  int phase_fallback;   /* RuntimePolicy.phase_fallback */
  int prefix_cap;       /* RuntimePolicy.prefix_cap */
  int replan_size;      /* RuntimePolicy.replan_size */
} sf_verify_cfg_t;

/* VerifierReport (verifier.py:53-62) outputs, all device pointers. For batched
 * entry points each array gains a leading env dimension. */
typedef struct {
  void* draft;            /* [H*D]            (may be NULL) */
  void* reconstructed;    /* [K*H*D]          (may be NULL) */
  void* distances;        /* [K*H]            (may be NULL) */
  int* branch_prefixes;   /* [K]              */
  int* result;            /* [SF_RESULT_WORDS] */
} sf_verify_out_t;

const char* sf_last_error(void);
int sf_version(void);
/* Number of kernels the library launched on this thread since the last reset. */
int64_t sf_launch_count(int reset);

/* Staging helpers for the host-facing API: async copy of `bytes` from a
 * (pinned) host buffer to the device on `stream`; copy back and synchronize
 * the stream. */
int sf_copy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int sf_copy_d2h_sync(void* dst, const void* src, size_t bytes, void* stream);

/* ------------------------------------------------------------------ tiny path
 * cfg1/cfg2: tanh-MLP draft + endpoint-parameterised MLP field.
 * One cluster-resident launch per round; weights stream from L2. */

/* Speculative round: propose (draft.py:57-61) + verify (verifier.py:109-150)
 * + fallback decision (runtime.py:286-320), fused in ONE kernel.
 * If `draft_net` is NULL, `draft_in` holds the draft values [H*D] (the
 * reference's verify() given a chunk); otherwise `draft_in` holds the draft
 * features and the draft MLP runs on device. `eps` is the shared noise
 * (verifier.py:129) [H*D]. `emb` is the cached context (flowpolicy.py:38-50),
 * `state` the normalised robot state. Elements are float (SF_F32) or double
 * (SF_F64). */
int sf_tiny_flash_round(int precision, const sf_mlp_t* draft_net, const void* draft_in,
                        const sf_mlp_t* field_net, const void* emb, int emb_dim,
                        const void* state, int state_dim, const void* eps,
                        int horizon, int dim, int continuous_dims,
                        const sf_verify_cfg_t* cfg, const sf_verify_out_t* out, void* stream);

/* Full round: encode_context (flowpolicy.py:156-161) + integrate_flow
 * (flowpolicy.py:273-292), N Euler steps in ONE kernel. If `encoder` is NULL,
 * `enc_in` is the cached embedding itself [emb_dim]; otherwise it is the
 * encoder feature vector [encoder->sizes[0]] and emb = [features, MLP(features)].
 * `start` is the initial noise A^0 [H*D]. Outputs: chunk [H*D], emb_out
 * [emb_dim] (may be NULL), status[2] = {first non-finite step or -1,
 * 1 if the velocity (vs the state) was non-finite}. num_steps == 0 runs
 * encode_context only (field_net may then be NULL). */
int sf_tiny_full_round(int precision, const sf_mlp_t* encoder, const void* enc_in, int emb_dim,
                       const sf_mlp_t* field_net, const void* state, int state_dim,
                       const void* start, int horizon, int dim, int num_steps,
                       void* chunk_out, void* emb_out, int* status, void* stream);

/* Tanh-MLP forward of `rows` (<= 8) input rows (nets.forward, nets.py:90-107;
 * the draft's propose, draft.py:57-61): x [rows*n_in] -> out [rows*n_out]. */
int sf_tiny_mlp_forward(int precision, const sf_mlp_t* net, const void* x, int rows, void* out,
                        void* stream);

/* Field protocol evaluation of the tiny endpoint field for `rows` (<= 8) states
 * (VelocityField.evaluate, flowpolicy.py:203-209): x [rows*H*D], taus[rows]
 * (host), v = (net([x, tau, emb, state]) - x) / (1 - tau) -> velocity_out
 * [rows*H*D]; status[rows] = 1 where v is non-finite (may be NULL). */
int sf_tiny_field_eval(int precision, const sf_mlp_t* field_net, const void* x, const double* taus,
                       int rows, const void* emb, int emb_dim, const void* state, int state_dim,
                       int horizon, int dim, void* velocity_out, int* status, void* stream);

/* ----------------------------------------------------- field-agnostic pieces
 * For fields evaluated elsewhere (the reference's field protocol,
 * flowpolicy.py:249-261): the device does interpolation, reconstruction,
 * distances, prefix scan, gripper gate and decision. */

/* x_k = tau_k * draft + (1 - tau_k) * eps for every k (verifier.py:65-73); out [K*n].
 * `taus` is a HOST array of k doubles in [0, 1]. */
int sf_interpolate(int precision, const void* draft, const void* eps, const double* taus, int k,
                   int n, void* out, void* stream);

/* Given velocities v_k [K*H*D] at x_k: recon, distances, per-branch prefix,
 * min, gripper gate, decision (verifier.py:76-150, runtime.py:286-320). */
int sf_verify_epilogue(int precision, const void* draft, const void* eps, const void* velocity,
                       int horizon, int dim, int continuous_dims, const sf_verify_cfg_t* cfg,
                       const sf_verify_out_t* out, void* stream);

/* prefix_length (verifier.py:94-106) for `rows` independent distance rows [rows*h]. */
int sf_prefix_length(int precision, const void* distances, int rows, int h, double delta,
                     int* out, void* stream);

/* continuous_distances (actions.py:168-181): a,b [rows*dim] -> out [rows]. */
int sf_continuous_distances(int precision, const void* a, const void* b, int rows, int dim,
                            int continuous_dims, int metric, void* out, void* stream);

/* gripper_switch (actions.py:193-211) over `n_chunks` chunks [n_chunks*H*D]; out[0] = 0/1. */
int sf_gripper_switch(int precision, const void* values, int n_chunks, int horizon, int dim,
                      double current_sign, int window, int* out, void* stream);

/* One Euler update values += v / n with the finite check (flowpolicy.py:289-291);
 * status[0] set to `step` on the first non-finite result (caller inits to -1). */
int sf_euler_update(int precision, void* values, const void* velocity, int count, int n, int step,
                    int* status, void* stream);

/* Device-side round bookkeeping of a batch of independent envs
 * (run_episode, runtime.py:238-320), after a batched flash attempt:
 *   forced = PF > 0 && fsr[e] >= PF;  use_flash = mode_flash && has_cache[e] && !forced
 *   !use_flash            -> path FULL (PERIODIC if forced in flash mode), planned = R
 *   flash rejected/phase  -> path from result[e] (SF_RES_PATH), planned = R
 *   flash accepted        -> planned = result[e][SF_RES_PLANNED], fsr[e] += 1
 *   every full round      -> fsr[e] = 0, has_cache[e] = 1
 * Envs needing the full (Euler) path are compacted in env order into
 * fb_idx[0 .. *fb_count) (one CTA, block scan: deterministic), so the Euler
 * denoise runs on that bucket only (sf_ae_denoise_envs with env_map = fb_idx).
 * result: [n_envs][SF_RESULT_WORDS] device words of the flash round (ignored
 * where use_flash is 0); fsr, has_cache: [n_envs] in/out; path, planned,
 * fb_idx: [n_envs] out; fb_count: [1] out. All device pointers. */
int sf_replan_update(int n_envs, const int* result, int* fsr, int* has_cache, int mode_flash,
                     int periodic_refresh, int replan_size, int* path, int* planned, int* fb_idx,
                     int* fb_count, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPECFLOW_B200_H */
