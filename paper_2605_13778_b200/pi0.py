"""pi0-scale Action Expert on the device (BASELINE configs 3-5).

The reference substitutes MLPs for the Action Expert; this is
the builder-defined pi0-scale field: 18 layers, width 1024, 8
query heads x 256 sharing one KV head (MQA), GeGLU 4096, RMSNorm, RoPE,
attending to a per-env VLM prefix KV cache (800 tokens) with the paper's
block mask. It honours the reference's field protocol
(``evaluate(values, tau, cache, state)``, ``horizon``, ``dim``, ``layout``,
``eval_count`` — flowpolicy.py:249-261), so the drop-in ``verify`` /
``integrate_flow`` dispatch to its fused device chains:

* ``device_verify``  -> ``sf_ae_verify`` (embed -> 18 x [QKV GEMM+RoPE, MQA
  attention, O GEMM, GeGLU GEMM, down GEMM] -> head GEMM -> verify
  epilogue), one CUDA graph with programmatic dependent launch;
* ``device_denoise`` -> ``sf_ae_denoise`` (N Euler steps in one graph).

Weights are random-init with a counter-based generator shared bit-for-bit with
``oracle/pi0_oracle.py`` and stored in the kernels' layouts (q/k rows paired
for RoPE, gate/up rows interleaved).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi, _device
from .actions import ChannelLayout

SF_AE_GRAPH, SF_AE_PDL, SF_AE_FP32 = 1, 2, 4
TID_A_W, TID_S_W, TID_T1_W, TID_T2_W, TID_OUT_W = 1, 2, 3, 4, 5
TID_DRAFT_BASE = 20
TID_LAYER_BASE = 100
TID_KV_BASE = 10000


@dataclass(frozen=True)
class AEConfig:
    width: int = 1024
    layers: int = 18
    q_heads: int = 8
    head_dim: int = 256
    mlp: int = 4096
    action_dim: int = 32
    state_dim: int = 32
    horizon: int = 50
    prefix_len: int = 800
    rope_base: float = 10000.0
    eps: float = 1e-6
    temb_min_period: float = 4e-3
    temb_max_period: float = 4.0
    draft_in: int = 64       # draft MLP observation features (0 disables the draft)
    draft_hidden: int = 1024

    @property
    def seg_len(self) -> int:
        return 1 + self.horizon

    def n_params(self) -> int:
        W, nq = self.width, self.q_heads * self.head_dim
        per_layer = (nq + 2 * self.head_dim) * W + W * nq + 2 * self.mlp * W + W * self.mlp
        io = (W * self.action_dim + W) + (W * self.state_dim + W) + 2 * (W * W + W) + \
            (self.action_dim * W + self.action_dim)
        return self.layers * per_layer + io

    def weight_bytes_streamed(self) -> int:
        """bf16 bytes of the per-layer GEMM weights + head read per forward."""
        W, nq = self.width, self.q_heads * self.head_dim
        per_layer = (nq + 2 * self.head_dim) * W + W * nq + 2 * self.mlp * W + W * self.mlp
        return 2 * (self.layers * per_layer + self.action_dim * W)

    def kv_bytes(self) -> int:
        return 2 * 2 * self.layers * self.prefix_len * self.head_dim


PI0 = AEConfig()


class _AeConfigC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("width", "layers", "q_heads", "head_dim", "mlp",
                                            "action_dim", "state_dim", "horizon", "prefix_len")] + \
               [("eps", ctypes.c_float), ("temb_min_period", ctypes.c_float),
                ("temb_max_period", ctypes.c_float), ("draft_in", ctypes.c_int),
                ("draft_hidden", ctypes.c_int)]


_MAXL = 32


class _AeWeightsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("a_w", "a_b", "s_w", "s_b", "t1_w", "t1_b", "t2_w",
                                               "t2_b", "out_w", "out_b")] + \
               [("qkv", ctypes.c_void_p * _MAXL), ("o", ctypes.c_void_p * _MAXL),
                ("gu", ctypes.c_void_p * _MAXL), ("down", ctypes.c_void_p * _MAXL),
                ("rope", ctypes.c_void_p), ("draft_w", ctypes.c_void_p * 3),
                ("draft_b", ctypes.c_void_p * 3)]


def _fill(t: torch.Tensor, seed: int, tid: int, std: float) -> torch.Tensor:
    _capi.check(_capi.lib().sf_fill_hash_uniform(
        t.data_ptr(), 1 if t.dtype == torch.bfloat16 else 0, t.numel(), seed, tid, std,
        torch.cuda.current_stream().cuda_stream), "init")
    return t


def rope_table(cfg: AEConfig, max_pos: int) -> np.ndarray:
    half = cfg.head_dim // 2
    inv = cfg.rope_base ** (-np.arange(half, dtype=np.float64) * 2.0 / cfg.head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)


def qkv_row_perm(cfg: AEConfig) -> torch.Tensor:
    """device row -> natural row: per head, rows (2i, 2i+1) = dims (i, i+128)."""
    hd, half = cfg.head_dim, cfg.head_dim // 2
    perm = []
    for head in range(cfg.q_heads + 1):  # q heads, then the k head
        base = head * hd
        for i in range(half):
            perm += [base + i, base + i + half]
    base = (cfg.q_heads + 1) * hd
    perm += list(range(base, base + hd))  # v rows unchanged
    return torch.tensor(perm, dtype=torch.long)


def gu_row_perm(cfg: AEConfig) -> torch.Tensor:
    """device row -> natural row: rows (2i, 2i+1) = (gate_i, up_i)."""
    idx = torch.arange(cfg.mlp)
    return torch.stack([idx, idx + cfg.mlp], dim=1).reshape(-1)


class ActionExpert:
    """Device-resident pi0-scale Action Expert + prefix KV pool (field protocol)."""

    def __init__(self, cfg: AEConfig = PI0, seed: int = 0, n_envs: int = 1, kv_seed: int = 1,
                 layout: ChannelLayout | None = None, std: float = 0.02,
                 flags: int = SF_AE_GRAPH | SF_AE_PDL, env_offset: int = 0,
                 draft_gripper_bias: float = 0.0, precision: str = "bf16"):
        """precision "bf16": tcgen05 kernels, bf16 activations / fp32 accumulation
        (the performance path); "fp32": verify / denoise run the fp32 mode
        (SF_AE_FP32: fp32 activations and FMA accumulation on CUDA cores, the
        north star's 1e-5 parity mode). Weights and prefix KV are bf16 in both."""
        if precision not in ("bf16", "fp32"):
            raise ValueError(f"unknown precision {precision!r}")
        if precision == "fp32":
            flags |= SF_AE_FP32
        self.precision = precision
        self.cfg = cfg
        self.horizon = cfg.horizon
        self.dim = cfg.action_dim
        self.layout = layout or ChannelLayout(cfg.action_dim - 1, 0)
        if self.layout.dim != cfg.action_dim:
            raise ValueError("layout does not match action_dim")
        self.eval_count = 0
        self.flags = flags
        self.seed = seed
        dev = _device.device()
        W, nq, L = cfg.width, cfg.q_heads * cfg.head_dim, cfg.layers
        f32, b16 = torch.float32, torch.bfloat16
        self._keep = []

        def mk(shape, dtype, tid, s=std):
            t = _fill(torch.empty(shape, dtype=dtype, device=dev), seed, tid, s)
            self._keep.append(t)
            return t

        def zeros(n):
            t = torch.zeros(n, dtype=f32, device=dev)
            self._keep.append(t)
            return t

        w = _AeWeightsC()
        w.a_w = mk((W, cfg.action_dim), f32, TID_A_W).data_ptr()
        w.a_b = zeros(W).data_ptr()
        w.s_w = mk((W, cfg.state_dim), f32, TID_S_W).data_ptr()
        w.s_b = zeros(W).data_ptr()
        w.t1_w = mk((W, W), f32, TID_T1_W).data_ptr()
        w.t1_b = zeros(W).data_ptr()
        w.t2_w = mk((W, W), f32, TID_T2_W).data_ptr()
        w.t2_b = zeros(W).data_ptr()
        w.out_w = mk((cfg.action_dim, W), b16, TID_OUT_W).data_ptr()
        w.out_b = zeros(cfg.action_dim).data_ptr()
        pq = qkv_row_perm(cfg).to(dev)
        pg = gu_row_perm(cfg).to(dev)
        for l in range(L):
            b = TID_LAYER_BASE + 4 * l
            qkv_nat = _fill(torch.empty((nq + 2 * cfg.head_dim, W), dtype=b16, device=dev), seed, b, std)
            qkv = qkv_nat.index_select(0, pq).contiguous()
            del qkv_nat
            gu_nat = _fill(torch.empty((2 * cfg.mlp, W), dtype=b16, device=dev), seed, b + 2, std)
            gu = gu_nat.index_select(0, pg).contiguous()
            del gu_nat
            o = mk((W, nq), b16, b + 1)
            down = mk((W, cfg.mlp), b16, b + 3)
            self._keep += [qkv, gu]
            w.qkv[l], w.o[l], w.gu[l], w.down[l] = (qkv.data_ptr(), o.data_ptr(), gu.data_ptr(),
                                                    down.data_ptr())
        rope = torch.from_numpy(rope_table(cfg, cfg.prefix_len + cfg.seg_len)).to(dev)
        self._keep.append(rope)
        w.rope = rope.data_ptr()
        if cfg.draft_in > 0:
            # tanh MLP draft [draft_in -> hid -> hid -> H*D] (draft.py:29-61 at pi0 scale)
            hid, hdd = cfg.draft_hidden, cfg.horizon * cfg.action_dim
            shapes = ((hid, cfg.draft_in), (hid, hid), (hdd, hid))
            for i, shp in enumerate(shapes):
                w.draft_w[i] = mk(shp, b16, TID_DRAFT_BASE + i, float(np.sqrt(1.0 / shp[1]))).data_ptr()
                bias = zeros(shp[0])
                if i == 2 and draft_gripper_bias:
                    # one-signed gripper column (last channel of every row): a
                    # draft that holds the gripper state, so phase fallbacks come
                    # from the current sign, not from random draft signs
                    bias.view(cfg.horizon, cfg.action_dim)[:, -1] = draft_gripper_bias
                w.draft_b[i] = bias.data_ptr()
        c = _AeConfigC(cfg.width, cfg.layers, cfg.q_heads, cfg.head_dim, cfg.mlp, cfg.action_dim,
                       cfg.state_dim, cfg.horizon, cfg.prefix_len, cfg.eps, cfg.temb_min_period,
                       cfg.temb_max_period, cfg.draft_in, cfg.draft_hidden)
        self._cfg_c, self._w_c = c, w
        h = ctypes.c_void_p()
        _capi.check(_capi.lib().sf_ae_create(ctypes.byref(c), ctypes.byref(w), ctypes.byref(h)),
                    "ae create")
        self._h = h
        self.n_envs = 0
        self.set_prefix_pool(n_envs, kv_seed, env_offset)

    # ---------------------------------------------------------- prefix KV
    def set_prefix_pool(self, n_envs: int, kv_seed: int = 1, env_offset: int = 0):
        """Random-init prefix KV for envs [env_offset, env_offset + n_envs)
        (stand-in for the VLM prefill; same values as oracle make_prefix_kv)."""
        cfg, dev = self.cfg, _device.device()
        L, P, hd = cfg.layers, cfg.prefix_len, cfg.head_dim
        self.k_prefix = torch.empty((L, n_envs, P, hd), dtype=torch.bfloat16, device=dev)
        self.vt_prefix = torch.empty((L, n_envs, hd, P), dtype=torch.bfloat16, device=dev)
        for e in range(n_envs):
            for l in range(L):
                t = TID_KV_BASE + 2 * ((env_offset + e) * L + l)
                _fill(self.k_prefix[l, e], kv_seed, t, 1.0)
                _fill(self.vt_prefix[l, e], kv_seed, t + 1, 1.0)
        _capi.check(_capi.lib().sf_ae_set_prefix(self._h, self.k_prefix.data_ptr(),
                                                 self.vt_prefix.data_ptr(), n_envs), "prefix")
        self.n_envs = n_envs
        self.kv_seed = kv_seed

    def bind_prefix(self, k_pool: torch.Tensor, vt_pool: torch.Tensor):
        """Attend to an externally produced prefix KV pool (e.g. the output of
        VLMPrefill.prefill: K [L, E, P, 256], V^T [L, E, 256, P] bf16)."""
        cfg = self.cfg
        L, E, P, hd = k_pool.shape
        if (L, P, hd) != (cfg.layers, cfg.prefix_len, cfg.head_dim) or tuple(vt_pool.shape) != (L, E, hd, P):
            raise ValueError("prefix pool shape does not match the Action Expert config")
        self.k_prefix, self.vt_prefix = k_pool, vt_pool
        _capi.check(_capi.lib().sf_ae_set_prefix(self._h, k_pool.data_ptr(), vt_pool.data_ptr(), E),
                    "prefix")
        self.n_envs = E

    def refresh_prefix(self, stream=None):
        """Re-derive the attention's block images of the bound pool after it
        was rewritten in place (context refresh into ``k_prefix`` /
        ``vt_prefix``), ordered on ``stream`` after that write."""
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _capi.check(_capi.lib().sf_ae_refresh_prefix(self._h, s), "refresh prefix")

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _capi.lib().sf_ae_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # ----------------------------------------------------- device batched API
    def verify_batch(self, cfg, draft: torch.Tensor, eps: torch.Tensor, state: torch.Tensor,
                     signs: torch.Tensor | None = None, current_sign: float = -1.0,
                     phase_fallback=True, prefix_cap=True, replan_size=12, outputs=None,
                     stream=None):
        """Device tensors in, device tensors out (no sync). draft/eps [B,H,D] f32,
        state [B,S] f32, signs [B] f32. Returns (recon, dist, branch, result)."""
        from .verifier import make_cfg

        B = draft.shape[0]
        K = len(cfg.timesteps)
        dev = draft.device
        if outputs is None:
            outputs = (torch.empty((B, K, self.horizon, self.dim), dtype=torch.float32, device=dev),
                       torch.empty((B, K, self.horizon), dtype=torch.float32, device=dev),
                       torch.empty((B, K), dtype=torch.int32, device=dev),
                       torch.empty((B, _capi.SF_RESULT_WORDS), dtype=torch.int32, device=dev))
        recon, dist, branch, result = outputs
        c = make_cfg(cfg, current_sign, phase_fallback, prefix_cap, replan_size)
        out = _capi.SfVerifyOut(None, recon.data_ptr() if recon is not None else None,
                                dist.data_ptr() if dist is not None else None, branch.data_ptr(),
                                result.data_ptr())
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _capi.check(_capi.lib().sf_ae_verify(
            self._h, B, ctypes.byref(c), draft.data_ptr(), eps.data_ptr(), state.data_ptr(),
            signs.data_ptr() if signs is not None else None, ctypes.byref(out), self.flags, s),
            "ae verify")
        return outputs

    def flash_batch(self, cfg, obs: torch.Tensor, eps: torch.Tensor, state: torch.Tensor,
                    signs: torch.Tensor | None = None, current_sign: float = -1.0,
                    phase_fallback=True, prefix_cap=True, replan_size=12, outputs=None,
                    stream=None):
        """Speculative round for B envs in one graph: draft MLP on obs [B, F]
        -> verify -> gate/decision. Returns (draft, recon, dist, branch, result)."""
        from .verifier import make_cfg

        B = obs.shape[0]
        K = len(cfg.timesteps)
        dev = obs.device
        if outputs is None:
            outputs = (torch.empty((B, self.horizon, self.dim), dtype=torch.float32, device=dev),
                       torch.empty((B, K, self.horizon, self.dim), dtype=torch.float32, device=dev),
                       torch.empty((B, K, self.horizon), dtype=torch.float32, device=dev),
                       torch.empty((B, K), dtype=torch.int32, device=dev),
                       torch.empty((B, _capi.SF_RESULT_WORDS), dtype=torch.int32, device=dev))
        draft, recon, dist, branch, result = outputs
        c = make_cfg(cfg, current_sign, phase_fallback, prefix_cap, replan_size)
        out = _capi.SfVerifyOut(draft.data_ptr(), recon.data_ptr() if recon is not None else None,
                                dist.data_ptr() if dist is not None else None, branch.data_ptr(),
                                result.data_ptr())
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _capi.check(_capi.lib().sf_ae_flash_round(
            self._h, B, ctypes.byref(c), obs.data_ptr(), eps.data_ptr(), state.data_ptr(),
            signs.data_ptr() if signs is not None else None, ctypes.byref(out), self.flags, s),
            "ae flash round")
        return outputs

    def time_op(self, n_envs: int, k: int, op: int, iters: int, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _capi.check(_capi.lib().sf_ae_time_op(self._h, n_envs, k, op, iters, s), "time op")

    def denoise_batch(self, start: torch.Tensor, state: torch.Tensor, n_steps: int,
                      chunk: torch.Tensor | None = None, status: torch.Tensor | None = None,
                      stream=None):
        B = start.shape[0]
        dev = start.device
        chunk = torch.empty_like(start) if chunk is None else chunk
        status = torch.empty((B, 2), dtype=torch.int32, device=dev) if status is None else status
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _capi.check(_capi.lib().sf_ae_denoise(self._h, B, n_steps, start.data_ptr(),
                                              state.data_ptr(), chunk.data_ptr(), status.data_ptr(),
                                              self.flags, s), "ae denoise")
        return chunk, status

    def denoise_envs(self, env_map: torch.Tensor, start: torch.Tensor, state: torch.Tensor,
                     n_steps: int, chunk: torch.Tensor | None = None,
                     status: torch.Tensor | None = None, stream=None):
        """Euler full path on a compacted batch: row e attends to prefix-KV pool
        slot env_map[e] (int32 device tensor)."""
        B = start.shape[0]
        dev = start.device
        chunk = torch.empty_like(start) if chunk is None else chunk
        status = torch.empty((B, 2), dtype=torch.int32, device=dev) if status is None else status
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _capi.check(_capi.lib().sf_ae_denoise_envs(self._h, B, env_map.data_ptr(), n_steps,
                                                   start.data_ptr(), state.data_ptr(),
                                                   chunk.data_ptr(), status.data_ptr(), self.flags, s),
                    "ae denoise envs")
        return chunk, status

    def velocity_batch(self, x: torch.Tensor, taus, state: torch.Tensor) -> torch.Tensor:
        """x [B, R, H, D] f32 -> v [B, R, H, D] (field protocol, batched)."""
        B, R = x.shape[0], x.shape[1]
        out = torch.empty_like(x)
        _capi.check(_capi.lib().sf_ae_velocity(
            self._h, B, R, x.data_ptr(), _capi.host_doubles(list(taus)), state.data_ptr(),
            out.data_ptr(), torch.cuda.current_stream().cuda_stream), "ae velocity")
        return out

    # --------------------------------------------- reference field protocol
    def _env_of(self, cache) -> int:
        env = int(cache.kv) if cache is not None and cache.kv is not None else 0
        if not 0 <= env < self.n_envs:
            raise ValueError(f"cache refers to prefix env {env}, pool has {self.n_envs}")
        return env

    def evaluate(self, values, tau, cache, state) -> np.ndarray:
        """v(A, tau) for one chunk (flowpolicy.py:203-209 protocol)."""
        self.eval_count += 1
        if self._env_of(cache) != 0:
            raise ValueError("single-chunk evaluation uses prefix env 0")
        dev = _device.device()
        x = torch.as_tensor(np.asarray(values, np.float32)).to(dev).reshape(1, 1, self.horizon, self.dim)
        st = torch.as_tensor(np.asarray(state, np.float32)).to(dev).reshape(1, -1)
        return self.velocity_batch(x, [tau], st)[0, 0].double().cpu().numpy()

    def device_verify(self, draft, cache, state, cfg, eps, current_sign, noise_seed):
        """The reference-facing plugin call (verifier.verify on this field):
        numpy in, numpy out. Inputs go up in ONE pinned copy, recon /
        distances / branch prefixes / result words come back in ONE copy
        (``_device.Staging``), around one ``sf_ae_verify`` graph launch."""
        from .verifier import VerifierReport, make_cfg

        if self._env_of(cache) != 0:
            raise ValueError("single-env verify uses prefix env 0")
        H, D = self.horizon, self.dim
        K = len(cfg.timesteps)
        vals = np.asarray(draft.values, np.float64)
        st_in = np.asarray(state, np.float64).ravel()
        stg = _device.Staging.get("ae_verify", 2 * H * D + st_in.size, K * H * D + K * H,
                                  K + _capi.SF_RESULT_WORDS, torch.float32)
        p_d, p_e, p_s = stg.upload([vals, np.asarray(eps, np.float64), st_in])
        out = stg.extra.get(("vout", K))
        if out is None:
            out = stg.extra[("vout", K)] = _capi.SfVerifyOut(
                None, stg.out_ptr(0), stg.out_ptr(K * H * D), stg.word_ptr(_capi.SF_RESULT_WORDS),
                stg.word_ptr(0))
        c = make_cfg(cfg, current_sign)
        _capi.check(_capi.lib().sf_ae_verify(self._h, 1, ctypes.byref(c), p_d, p_e, p_s, None,
                                             ctypes.byref(out), self.flags, _device.stream_ptr()), "ae verify")
        v, words = stg.download(K * H * D + K * H, K + _capi.SF_RESULT_WORDS)
        res = words[:_capi.SF_RESULT_WORDS]
        if int(res[_capi.RES_NONFINITE]) >= 0:
            raise FloatingPointError(
                f"velocity produced non-finite values at tau={cfg.timesteps[int(res[_capi.RES_NONFINITE])]}")
        return VerifierReport(
            reconstructed=v[:K * H * D].reshape(K, H, D), distances=v[K * H * D:].reshape(K, H),
            branch_prefixes=tuple(int(x) for x in words[_capi.SF_RESULT_WORDS:]),
            prefix=int(res[_capi.RES_PREFIX]), gripper_switch_detected=bool(res[_capi.RES_SWITCH]),
            shared_noise_seed=noise_seed, decision=_capi.PATH_CODES[int(res[_capi.RES_PATH])],
            planned=int(res[_capi.RES_PLANNED]))

    def device_denoise(self, cache, state, start, n) -> np.ndarray:
        """integrate_flow on this field (plugin call): one pinned upload of the
        start noise + state, one ``sf_ae_denoise`` launch, one readback of the
        chunk and the status words."""
        if self._env_of(cache) != 0:
            raise ValueError("single-env denoise uses prefix env 0")
        self.eval_count += n
        H, D = self.horizon, self.dim
        st_in = np.asarray(state, np.float64).ravel()
        stg = _device.Staging.get("ae_denoise", H * D + st_in.size, H * D, 2, torch.float32)
        p_a, p_s = stg.upload([np.asarray(start, np.float64), st_in])
        _capi.check(_capi.lib().sf_ae_denoise(self._h, 1, n, p_a, p_s, stg.out_ptr(0), stg.word_ptr(0),
                                              self.flags, _device.stream_ptr()), "ae denoise")
        chunk, sv = stg.download(H * D, 2)
        if sv[0] >= 0:
            step = int(sv[0])
            if sv[1]:
                raise FloatingPointError(f"velocity produced non-finite values at tau={step / n}")
            raise FloatingPointError(f"denoising diverged at step {step} (tau={step / n})")
        return chunk.reshape(H, D)


class BatchedReplanner:
    """Device-side replanning rounds for B independent envs (run_episode,
    runtime.py:219-334, minus the conveyor), ONE graph launch per round with no
    host synchronisation (``sf_ae_replan_round``): the batched flash attempt
    (draft + K-branch verify + gate + decision for every env), the round
    bookkeeping on the device (periodic-refresh counter, path codes, planned
    prefix with the cap, fallback compaction), then a graph SWITCH node picks
    the smallest pre-captured Euler bucket (powers of two up to 64, then
    multiples of 64) holding the fallback envs and runs the N-step full path
    on it (bucket rows gathered / scattered on the device, each attending to
    its env's prefix KV). A final kernel flags non-finite chunks (planned = 0;
    the reference raises FloatingPointError, flowpolicy.py:290 /
    verifier.py:89), computes ``switch_in_executed`` for accepted rounds
    (runtime.py:321-323) and destandardizes the chunk when a Standardizer is
    given (actions.py:139-144, runtime.py:325).

    The speculative attempt itself runs only for the envs that make one this
    round (a cached context and no forced periodic refresh, runtime.py:242-253):
    they are compacted on the device into the smallest pre-captured flash
    bucket (powers of two up to 32, then multiples of 32) by a second SWITCH,
    and a round of full rounds only runs no attempt at all.

    ``round`` returns device tensors (chunk [B, H, D] standardized, path codes
    ``_capi.SF_PATH_*``, planned, branch prefixes [B, K], flash result words
    [B, 8]; branch prefixes and result words 0-4 are -1 for envs without an
    attempt this round); ``chunk_raw``,
    ``switch_in_executed``, ``nonfinite`` and ``n_fallback`` are attributes
    updated by the same launch."""

    def __init__(self, ae: ActionExpert, n_envs: int, vcfg, replan_size: int = 12,
                 periodic_refresh: int = 2, phase_fallback: bool = True, prefix_cap: bool = True,
                 flash: bool = True, num_steps: int = 10, standardizer=None):
        if n_envs > ae.n_envs:
            raise ValueError(f"{n_envs} envs but the prefix pool holds {ae.n_envs}")
        if replan_size < 1:
            raise ValueError("replan_size must be >= 1")
        if periodic_refresh < 0:
            raise ValueError("periodic_refresh must be >= 0")
        from .verifier import make_cfg

        self.ae, self.n, self.vcfg = ae, n_envs, vcfg
        self.replan_size, self.periodic_refresh = replan_size, periodic_refresh
        self.phase_fallback, self.prefix_cap, self.flash = phase_fallback, prefix_cap, flash
        self.num_steps = num_steps
        dev = _device.device()
        i32 = dict(dtype=torch.int32, device=dev)
        H, D, K = ae.horizon, ae.dim, len(vcfg.timesteps)
        self.fsr = torch.zeros(n_envs, **i32)        # flash rounds since the last full round
        self.has_cache = torch.zeros(n_envs, **i32)  # a full round has produced a context
        self.chunk = torch.empty((n_envs, H, D), dtype=torch.float32, device=dev)
        self.chunk_raw = torch.empty_like(self.chunk) if standardizer is not None else None
        self.path = torch.empty(n_envs, **i32)
        self.planned = torch.empty(n_envs, **i32)
        self.switch_in_executed = torch.empty(n_envs, **i32)
        self.nonfinite = torch.empty(n_envs, **i32)
        self.branch = torch.empty((n_envs, K), **i32)
        self.result = torch.empty((n_envs, _capi.SF_RESULT_WORDS), **i32)
        self.n_fallback = torch.zeros(1, **i32)
        self._std = None
        if standardizer is not None:
            self._std = (torch.as_tensor(np.asarray(standardizer.mean, np.float32)).to(dev),
                         torch.as_tensor(np.asarray(standardizer.std, np.float32)).to(dev))
        self._cfg = make_cfg(vcfg, -1.0, phase_fallback, prefix_cap, replan_size)
        self._pol = _capi.SfReplanPolicy(int(bool(flash)), periodic_refresh, num_steps,
                                         self._std[0].data_ptr() if self._std else None,
                                         self._std[1].data_ptr() if self._std else None)
        self._out = _capi.SfReplanOut(
            self.chunk.data_ptr(), self.chunk_raw.data_ptr() if self.chunk_raw is not None else None,
            self.path.data_ptr(), self.planned.data_ptr(), self.switch_in_executed.data_ptr(),
            self.nonfinite.data_ptr(), self.branch.data_ptr(), self.result.data_ptr(),
            self.n_fallback.data_ptr())
        self.round_index = 0
        # kernels of the selected Euler bucket body (gather, status init, N x
        # [embed, layers x (qkv, attention, o, gate/up, down), head, update], scatter)
        L = ae.cfg.layers
        self.body_kernels = 3 + num_steps * ((9 * L + 2) + 2 if ae.precision == "fp32" else 3 + 5 * L)

    def kernel_counts(self):
        """(fixed, flash verify, Euler body, largest flash bucket below n) of
        the last round's graph: a round launches `fixed` kernels, plus the
        flash verify's (+2 gather / scatter when the attempting envs fit a
        bucket <= the last value) when any env attempted, plus the Euler
        body's when any env ran the full path."""
        out = (ctypes.c_int * 4)()
        _capi.check(_capi.lib().sf_ae_replan_kernels(self.ae._h, out), "replan kernels")
        return tuple(out)

    def round(self, obs: torch.Tensor, eps_verify: torch.Tensor, eps_denoise: torch.Tensor,
              state: torch.Tensor, signs: torch.Tensor, stream=None):
        n = self.n
        for name, t, shape in (("obs", obs, (n, self.ae.cfg.draft_in)),
                               ("eps_verify", eps_verify, (n, self.ae.horizon, self.ae.dim)),
                               ("eps_denoise", eps_denoise, (n, self.ae.horizon, self.ae.dim)),
                               ("state", state, (n, self.ae.cfg.state_dim)), ("signs", signs, (n,))):
            if tuple(t.shape) != shape or t.dtype != torch.float32 or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous float32 tensor of shape {shape}")
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _capi.check(_capi.lib().sf_ae_replan_round(
            self.ae._h, n, ctypes.byref(self._cfg), ctypes.byref(self._pol), obs.data_ptr(),
            eps_verify.data_ptr(), eps_denoise.data_ptr(), state.data_ptr(), signs.data_ptr(),
            self.fsr.data_ptr(), self.has_cache.data_ptr(), ctypes.byref(self._out), self.ae.flags, s),
            "replan round")
        self.round_index += 1
        return self.chunk, self.path, self.planned, self.branch, self.result


# ---------------------------------------------------------------- VLM prefill

@dataclass(frozen=True)
class VLMConfig:
    """Gemma-2B-style prefix encoder (context refresh)."""
    width: int = 2048
    layers: int = 18
    q_heads: int = 8
    head_dim: int = 256
    mlp: int = 16384
    prefix_len: int = 800
    eps: float = 1e-6
    rope_base: float = 10000.0


class _VlmConfigC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("width", "layers", "q_heads", "head_dim", "mlp",
                                            "prefix_len")] + [("eps", ctypes.c_float)]


class _VlmWeightsC(ctypes.Structure):
    _fields_ = [("qkv", ctypes.c_void_p * _MAXL), ("o", ctypes.c_void_p * _MAXL),
                ("gu", ctypes.c_void_p * _MAXL), ("down", ctypes.c_void_p * _MAXL),
                ("rope", ctypes.c_void_p)]


TID_VLM_BASE = 1000


class VLMPrefill:
    """Context refresh at pi0 scale: token embeddings of the P prefix tokens
    per env -> the prefix KV pool the Action Expert attends to (the
    encode_context analogue, flowpolicy.py:156-161; runtime.py:166 refreshes
    the cache on every full round). Random-init weights from the shared
    counter-based initialiser (oracle/pi0_oracle.py make_vlm_weights)."""

    def __init__(self, cfg: VLMConfig = VLMConfig(), seed: int = 7, std: float = 0.02):
        self.cfg = cfg
        dev = _device.device()
        W, nq, L = cfg.width, cfg.q_heads * cfg.head_dim, cfg.layers
        b16 = torch.bfloat16
        self._keep = []
        w = _VlmWeightsC()
        pq, pg = qkv_row_perm(cfg).to(dev), gu_row_perm(cfg).to(dev)
        for l in range(L):
            b = TID_VLM_BASE + 4 * l
            qkv = _fill(torch.empty((nq + 2 * cfg.head_dim, W), dtype=b16, device=dev), seed, b, std)
            qkv = qkv.index_select(0, pq).contiguous()
            gu = _fill(torch.empty((2 * cfg.mlp, W), dtype=b16, device=dev), seed, b + 2, std)
            gu = gu.index_select(0, pg).contiguous()
            o = _fill(torch.empty((W, nq), dtype=b16, device=dev), seed, b + 1, std)
            down = _fill(torch.empty((W, cfg.mlp), dtype=b16, device=dev), seed, b + 3, std)
            self._keep += [qkv, gu, o, down]
            w.qkv[l], w.o[l], w.gu[l], w.down[l] = (qkv.data_ptr(), o.data_ptr(), gu.data_ptr(),
                                                    down.data_ptr())
        rope = torch.from_numpy(rope_table(cfg, cfg.prefix_len)).to(dev)
        self._keep.append(rope)
        w.rope = rope.data_ptr()
        c = _VlmConfigC(W, L, cfg.q_heads, cfg.head_dim, cfg.mlp, cfg.prefix_len, cfg.eps)
        self._c, self._w = c, w
        h = ctypes.c_void_p()
        _capi.check(_capi.lib().sf_vlm_create(ctypes.byref(c), ctypes.byref(w), ctypes.byref(h)),
                    "vlm create")
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _capi.lib().sf_vlm_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def prefill(self, x: torch.Tensor, k_pool: torch.Tensor | None = None,
                vt_pool: torch.Tensor | None = None, stream=None, expert: "ActionExpert | None" = None):
        """x [E, P, W] f32 -> (k_pool [L, E, P, 256], vt_pool [L, E, 256, P]) bf16.
        ``expert``: an ActionExpert whose BOUND pool this prefill rewrites in
        place; its attention block images are refreshed on the same stream."""
        cfg = self.cfg
        E = x.shape[0]
        dev = x.device
        if k_pool is None:
            k_pool = torch.empty((cfg.layers, E, cfg.prefix_len, cfg.head_dim), dtype=torch.bfloat16,
                                 device=dev)
        if vt_pool is None:
            vt_pool = torch.empty((cfg.layers, E, cfg.head_dim, cfg.prefix_len), dtype=torch.bfloat16,
                                  device=dev)
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _capi.check(_capi.lib().sf_vlm_prefill(self._h, E, x.contiguous().data_ptr(), k_pool.data_ptr(),
                                               vt_pool.data_ptr(), s), "vlm prefill")
        if expert is not None:
            expert.refresh_prefix(s)
        return k_pool, vt_pool

