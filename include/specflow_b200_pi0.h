/*
 * specflow_b200 — pi0-scale Action Expert entry points (BASELINE configs 3-5).
 *
 * The reference has no pi0-scale model (SPEC.md:155 substitutes MLPs); these
 * entry points implement the reference's field protocol
 * (flowpolicy.py:249-261) and the verify / integrate_flow contracts
 * (verifier.py:109-150, flowpolicy.py:273-292) for the builder-defined Action
 * Expert (oracle/pi0_oracle.py). Same conventions as
 * specflow_b200.h. All array arguments are DEVICE pointers unless noted.
 */
#ifndef SPECFLOW_B200_PI0_H
#define SPECFLOW_B200_PI0_H

#include <stdint.h>

#include "specflow_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define SF_AE_MAX_LAYERS 32

#define SF_AE_GRAPH 1 /* capture/replay the round as a CUDA graph */
#define SF_AE_PDL 2   /* programmatic dependent launch between kernels */
#define SF_AE_FP32 4  /* fp32 mode: the layer stack + head of sf_ae_verify / sf_ae_denoise*
                         in fp32 activations with fp32 FMA accumulation (CUDA cores), the
                         north star's "1e-5 in an fp32 mode" parity mode (~10 ms / verify);
                         weights and prefix KV stay the model's bf16 values */

typedef struct {
  int width;       /* 1024 */
  int layers;      /* 18 */
  int q_heads;     /* 8 (one shared KV head, head_dim 256) */
  int head_dim;    /* 256 (fixed by the kernels) */
  int mlp;         /* 4096 (GeGLU) */
  int action_dim;  /* D = 32; gripper = last channel */
  int state_dim;   /* 32 */
  int horizon;     /* H = 50 (suffix = 1 state + H action tokens) */
  int prefix_len;  /* P = 800 prefix KV tokens */
  float eps;       /* RMSNorm epsilon */
  float temb_min_period, temb_max_period;
  int draft_in;     /* draft MLP input features (multiple of 64); 0 = no draft */
  int draft_hidden; /* draft MLP hidden width (multiple of 64) */
} sf_ae_config_t;

/* Device weights in DEVICE layout (see paper_2605_13778_b200/pi0.py):
 *  a_w [W, D] f32, a_b [W] f32      action_in
 *  s_w [W, S] f32, s_b [W] f32      state_proj
 *  t1_w, t2_w [W, W] f32, t1_b, t2_b [W] f32   time MLP
 *  out_w [D, W] bf16, out_b [D] f32 action head
 *  qkv[l] [(heads+2)*256, W] bf16   q/k rows interleaved (dim i, dim i+128)
 *  o[l] [W, heads*256] bf16
 *  gu[l] [2*mlp, W] bf16            rows interleaved (gate_i, up_i)
 *  down[l] [W, mlp] bf16
 *  rope [(P + 1 + H) * 128] float2 (cos, sin)
 *  draft_w[0..2] bf16 [hid, in], [hid, hid], [H*D, hid]; draft_b[0..2] f32
 *  (tanh MLP draft, draft.py:57-61 at pi0 scale) */
typedef struct {
  const void *a_w, *a_b, *s_w, *s_b, *t1_w, *t1_b, *t2_w, *t2_b, *out_w, *out_b;
  const void* qkv[SF_AE_MAX_LAYERS];
  const void* o[SF_AE_MAX_LAYERS];
  const void* gu[SF_AE_MAX_LAYERS];
  const void* down[SF_AE_MAX_LAYERS];
  const void* rope;
  const void* draft_w[3];
  const void* draft_b[3];
} sf_ae_weights_t;

/* The weight pointers are borrowed (device memory owned by the caller) and must
 * stay valid and unchanged for the handle's lifetime; the embedding weights
 * a_w / s_w are additionally copied once, transposed, at create time. */
int sf_ae_create(const sf_ae_config_t* cfg, const sf_ae_weights_t* weights, void** handle);
int sf_ae_destroy(void* handle);

/* Bind the prefix KV pool (the VLM prefill output, flowpolicy.py:38-50 cache):
 * k_prefix [L][n_envs][P][256] bf16, vt_prefix [L][n_envs][256][P] bf16. Env
 * e of a batched call attends to pool entry e. */
int sf_ae_set_prefix(void* handle, const void* k_prefix, const void* vt_prefix, int n_envs);

/* The attention reads per-64-key-block images of the bound pool, built by
 * sf_ae_set_prefix. After the bound pool is rewritten in place (a context
 * refresh: sf_vlm_prefill into the bound pool), call this on the stream of that
 * write to rebuild the images before the next verify / denoise. Async. */
int sf_ae_refresh_prefix(void* handle, void* stream);

/* Batched speculative verification (verifier.py:109-150 + runtime.py:286-320)
 * for n_envs envs: draft, eps [n_envs][H][D] f32, state [n_envs][S] f32,
 * signs [n_envs] f32 (NULL: cfg->current_sign). Outputs (each may be NULL
 * except branch_prefixes/result): reconstructed [n_envs][K][H][D] f32,
 * distances [n_envs][K][H] f32, branch_prefixes [n_envs][K], result
 * [n_envs][SF_RESULT_WORDS]. */
int sf_ae_verify(void* handle, int n_envs, const sf_verify_cfg_t* cfg, const float* draft,
                 const float* eps, const float* state, const float* signs,
                 const sf_verify_out_t* out, int flags, void* stream);

/* Batched speculative round = propose (draft MLP on obs [n_envs][draft_in]
 * f32, draft.py:57-61) + sf_ae_verify in ONE graph; out->draft receives the
 * draft [n_envs][H][D] f32 (runtime.py:173-198 flash_attempt). */
int sf_ae_flash_round(void* handle, int n_envs, const sf_verify_cfg_t* cfg, const float* obs,
                      const float* eps, const float* state, const float* signs,
                      const sf_verify_out_t* out, int flags, void* stream);

/* Run planned GEMM op `op` (0 .. 4*layers) of the (n_envs, k)
 * verify plan `iters` times back to back on `stream` — bench hook for the
 * per-kernel roofline. */
int sf_ae_time_op(void* handle, int n_envs, int k, int op, int iters, void* stream);

/* Per-kernel warm device times (us) of one eager verify round, launch order:
 * embed, layers x [qkv, attention, o, gate/up, down], head, epilogue. */
int sf_ae_profile_verify(void* handle, int n_envs, const sf_verify_cfg_t* cfg, const float* draft,
                         const float* eps, const float* state, float* times_us, int max_times,
                         int* n_times, void* stream);

/* Batched full path (flowpolicy.py:273-292): `start` = A^0 [n_envs][H][D];
 * chunk_out [n_envs][H][D]; status [n_envs][2] = {first non-finite step or -1,
 * 1 if a velocity was non-finite}. */
int sf_ae_denoise(void* handle, int n_envs, int num_steps, const float* start, const float* state,
                  float* chunk_out, int* status, int flags, void* stream);

/* sf_ae_denoise on a compacted batch: batch env e attends to prefix-KV pool
 * slot env_map[e] (device [n_envs], values in [0, n_prefix_envs); NULL =
 * identity). Used for the fallback bucket of a batched replanning round
 * (sf_replan_update). */
int sf_ae_denoise_envs(void* handle, int n_envs, const int* env_map, int num_steps, const float* start,
                       const float* state, float* chunk_out, int* status, int flags, void* stream);

/* ---- one batched replanning round on the device (run_episode, runtime.py:238-326) ----
 * ONE CUDA graph per (n_envs, verify cfg, policy): the speculative attempt for
 * every env (sf_ae_flash_round), the round bookkeeping (sf_replan_update:
 * periodic refresh, prefix cap, fallback compaction), then a device-selected
 * branch of a graph SWITCH node runs the N-step Euler full path on the
 * smallest pre-captured bucket that holds the fallback envs (buckets: powers
 * of two up to 64, then multiples of 64), gathers / scatters the compacted
 * rows on the device, and a final kernel marks non-finite chunks, computes
 * switch_in_executed for accepted rounds and destandardizes the chunk. No
 * host synchronisation inside the round. */
typedef struct {
  int mode_flash;        /* RuntimePolicy.mode == flash (0: every round is a full round) */
  int periodic_refresh;  /* PF (runtime.py:247-250) */
  int num_steps;         /* Euler steps of the full path (DenoiseConfig.num_steps) */
  const float* std_mean; /* [D] Standardizer mean / std (actions.py:139-144) for chunk_raw; */
  const float* std_std;  /* NULL: chunk_raw is not written */
} sf_replan_policy_t;

typedef struct {
  float* chunk;              /* [n][H][D] standardized chunk to execute (draft or full path) */
  float* chunk_raw;          /* [n][H][D] destandardize(chunk) (may be NULL) */
  int* path;                 /* [n] SF_PATH_* of the round */
  int* planned;              /* [n] actions to execute; 0 when the chunk is non-finite */
  int* switch_in_executed;   /* [n] accepted rounds: gripper switch in chunk[:planned] against the
                                env's current sign (runtime.py:321-323); 0 otherwise */
  int* nonfinite;            /* [n] 1: the chunk is non-finite (the reference raises
                                FloatingPointError, flowpolicy.py:290 / verifier.py:89) */
  int* branch_prefixes;      /* [n][K] of the flash attempt, -1 without one (may be NULL) */
  int* result;               /* [n][SF_RESULT_WORDS] of the flash attempt; words 0..SF_RES_NONFINITE
                                -1 for envs that made none this round (may be NULL) */
  int* n_fallback;           /* [1] envs that ran the full path (may be NULL) */
} sf_replan_out_t;

/* obs [n][draft_in], eps_verify / eps_denoise [n][H][D], state [n][S], signs [n]
 * (current gripper sign per env) f32; fsr / has_cache [n] int32 runner state
 * (in/out, flash_since_refresh and "has a cached context"). */
int sf_ae_replan_round(void* handle, int n_envs, const sf_verify_cfg_t* cfg,
                       const sf_replan_policy_t* policy, const float* obs, const float* eps_verify,
                       const float* eps_denoise, const float* state, const float* signs, int* fsr,
                       int* has_cache, const sf_replan_out_t* out, int flags, void* stream);

/* Kernel counts of the last sf_ae_replan_round graph (launch accounting; the
 * SWITCH bodies run only when selected on the device): out4 = {kernels of a
 * round with neither an attempt nor the full path, kernels of the flash
 * attempt's verify (+2 gather / scatter when the attempting envs fit a bucket
 * <= out4[3]), kernels of an Euler bucket body, largest flash bucket below n}. */
int sf_ae_replan_kernels(void* handle, int* out4);

/* Field protocol: velocities for n_envs x rows states x [..][rows][H][D] at
 * taus[rows] (HOST). */
int sf_ae_velocity(void* handle, int n_envs, int rows, const float* x, const double* taus,
                   const float* state, float* v_out, void* stream);

/* Counter-based initialiser shared bit-for-bit with oracle/pi0_oracle.py
 * (hash_uniform): dst[i] = U(-std*sqrt(3), std*sqrt(3)) from (seed, tid, i). */
int sf_fill_hash_uniform(void* dst, int is_bf16, int64_t n, uint64_t seed, uint64_t tid, double std,
                         void* stream);

/* ---- context refresh: VLM prefix prefill -> prefix KV pool ----
 * A Gemma-style decoder (8 query heads x 256 sharing one KV head, GeGLU MLP
 * `mlp`, RMSNorm gains folded into the weights, RoPE base 1e4) over the P
 * prefix tokens of each env with bidirectional prefix attention; layer l's K
 * and V are the Action Expert's prefix pool entries (flowpolicy.py:156-161
 * encode_context at pi0 scale). Weights use the Action Expert's device layout
 * (QKV rows interleaved for RoPE pairs, gate/up rows interleaved). */
typedef struct {
  int width;       /* 2048 for a Gemma-2B-style prefix encoder */
  int layers;
  int q_heads;     /* 8 */
  int head_dim;    /* 256 */
  int mlp;         /* 16384 */
  int prefix_len;  /* P (multiple of 16) */
  float eps;
} sf_vlm_config_t;

typedef struct {
  const void* qkv[SF_AE_MAX_LAYERS];   /* [8*256 + 2*256][W] bf16 */
  const void* o[SF_AE_MAX_LAYERS];     /* [W][8*256] bf16 */
  const void* gu[SF_AE_MAX_LAYERS];    /* [2*mlp][W] bf16 */
  const void* down[SF_AE_MAX_LAYERS];  /* [W][mlp] bf16 */
  const void* rope;                    /* [P][128] float2 (cos, sin) */
} sf_vlm_weights_t;

int sf_vlm_create(const sf_vlm_config_t* cfg, const sf_vlm_weights_t* weights, void** handle);
int sf_vlm_destroy(void* handle);
/* x [n_envs][P][W] f32 token embeddings -> k_pool [L][n_envs][P][256] bf16 and
 * vt_pool [L][n_envs][256][P] bf16 (the sf_ae_set_prefix layout). Async on
 * `stream`. */
int sf_vlm_prefill(void* handle, int n_envs, const float* x, void* k_pool, void* vt_pool, void* stream);

#ifdef __cplusplus
}
#endif

#endif
