"""Multi-step parallel verification (Alg. 1) on the device.

Drop-in for ``specflow.verifier`` (verifier.py:1-150): same names, signatures,
report type and exceptions. The K branches run as ONE batched field
evaluation, fused with interpolation, endpoint reconstruction, distances,
the warp-ballot prefix scan, the gripper gate and the fallback decision:

* MLP ``VelocityField`` (cfg1/cfg2): ``sf_tiny_flash_round`` (one launch);
* pi0-scale Action Expert: ``field.device_verify`` (tcgen05 chain, CUDA graph);
* any other field-protocol object: device interpolation, the field evaluated
  where it lives, then ``sf_verify_epilogue`` on the device.

The shared noise is drawn on the host from the caller's generator with the
reference's single ``standard_normal((H, D))`` call (verifier.py:129), so the
noise stream is bit-identical to the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _capi, _device
from .actions import STANDARDIZED, ActionChunk
from .flowpolicy import ConditioningCache, VelocityField, velocity


@dataclass(frozen=True)
class VerifierConfig:
    """Verification timesteps, threshold, metric, gripper window (verifier.py:29-50)."""

    timesteps: tuple = (1.0 / 3.0, 2.0 / 3.0)
    delta: float = 0.15
    metric: str = "l2"
    gripper_window: int | None = None

    def __post_init__(self) -> None:
        ts = tuple(float(t) for t in self.timesteps)
        if len(ts) == 0:
            raise ValueError("need at least one verification timestep")
        if not all(0.0 < t < 1.0 for t in ts):
            raise ValueError("verification timesteps must lie strictly inside (0, 1)")
        if any(nxt <= cur for cur, nxt in zip(ts, ts[1:])):
            raise ValueError("verification timesteps must be strictly increasing")
        if self.delta < 0.0:
            raise ValueError("delta must be non-negative")
        if self.metric not in _capi.SF_METRIC:
            raise ValueError(f"unknown metric {self.metric!r}")
        if len(ts) > _capi.SF_MAX_K:
            raise ValueError(f"at most {_capi.SF_MAX_K} verification timesteps are supported")
        object.__setattr__(self, "timesteps", ts)


@dataclass(frozen=True)
class VerifierReport:
    """verifier.py:53-62, plus the device's fallback decision for the round."""

    reconstructed: np.ndarray
    distances: np.ndarray
    branch_prefixes: tuple
    prefix: int
    gripper_switch_detected: bool
    shared_noise_seed: int | None = None
    decision: str | None = None  # runtime.py:286-291 path label under the policy used
    planned: int | None = None   # runtime.py:310, :319-320


_cfg_cache: dict = {}


def make_cfg(cfg: VerifierConfig, current_sign: float, phase_fallback: bool = True,
             prefix_cap: bool = True, replan_size: int = 12) -> "_capi.SfVerifyCfg":
    """C-ABI verifier config; memoised (configs are frozen, and building the
    ctypes struct costs several us on a ~0.1 ms round)."""
    key = (cfg, float(current_sign), bool(phase_fallback), bool(prefix_cap), int(replan_size))
    c = _cfg_cache.get(key)
    if c is None:
        if len(_cfg_cache) > 256:
            _cfg_cache.clear()
        c = _cfg_cache[key] = _make_cfg(cfg, current_sign, phase_fallback, prefix_cap, replan_size)
    return c


def _make_cfg(cfg: VerifierConfig, current_sign: float, phase_fallback: bool, prefix_cap: bool,
              replan_size: int) -> "_capi.SfVerifyCfg":
    c = _capi.SfVerifyCfg()
    c.k = len(cfg.timesteps)
    for i, t in enumerate(cfg.timesteps):
        c.taus[i] = t
    c.delta = float(cfg.delta)
    c.metric = _capi.SF_METRIC[cfg.metric]
    c.window = -1 if cfg.gripper_window is None else max(int(cfg.gripper_window), 0)
    c.current_sign = float(current_sign)
    c.phase_fallback = int(bool(phase_fallback))
    c.prefix_cap = int(bool(prefix_cap))
    c.replan_size = int(replan_size)
    return c


def interpolate(draft_values, eps, tau: float) -> np.ndarray:
    """tau * draft + (1 - tau) * eps on the device (verifier.py:65-73)."""
    a = np.asarray(draft_values, dtype=np.float64)
    e = np.asarray(eps, dtype=np.float64)
    if a.shape != e.shape:
        raise ValueError("draft and noise shapes differ")
    if not 0.0 <= tau <= 1.0:
        raise ValueError(f"tau={tau} outside [0, 1]")
    da, de = _device.to_dev(a), _device.to_dev(e)
    out = torch.empty_like(da)
    _capi.check(_capi.lib().sf_interpolate(_device.code(), da.data_ptr(), de.data_ptr(),
                                           _capi.host_doubles([tau]), 1, a.size, out.data_ptr(),
                                           _device.stream_ptr()), "interpolate")
    return _device.to_host(out).reshape(a.shape)


def reconstruct_endpoint(field, draft_values, eps, tau: float, cache: ConditioningCache,
                         state) -> np.ndarray:
    """x + (1 - tau) v(x, tau) at x = interpolate(...) (verifier.py:76-91)."""
    if not 0.0 < tau < 1.0:
        raise ValueError(f"tau={tau} outside (0, 1)")
    noisy = interpolate(draft_values, eps, tau)
    v = velocity(field, noisy, tau, cache, state)
    recon = _epilogue_recon(np.asarray(draft_values, np.float64), np.asarray(eps, np.float64), v,
                            tau)
    if not np.isfinite(recon).all():
        raise FloatingPointError(f"endpoint reconstruction at tau={tau} is non-finite")
    return recon


def _epilogue_recon(draft, eps, v, tau):
    h = draft.shape[0]
    d = draft.shape[1]
    cfg = VerifierConfig(timesteps=(tau,), delta=0.0)
    rep = _run_epilogue(draft, eps, v[None], cfg, -1.0, max(d - 1, 1), check=False)
    return rep[0].reshape(h, d)


def prefix_length(distances, delta: float) -> int:
    """Longest leading run of d <= delta: warp-ballot scan on device (verifier.py:94-106)."""
    d = np.asarray(distances, dtype=np.float64).ravel()
    if d.size == 0:
        return 0
    dd = _device.to_dev(d)
    out = torch.empty(1, dtype=torch.int32, device=dd.device)
    _capi.check(_capi.lib().sf_prefix_length(_device.code(), dd.data_ptr(), 1, d.size, float(delta),
                                             out.data_ptr(), _device.stream_ptr()), "prefix_length")
    return int(out.item())


def _decode(vals: np.ndarray, words: np.ndarray, k: int, h: int, d: int, seed, with_draft: bool):
    off = 0
    draft = None
    if with_draft:
        draft = vals[: h * d].reshape(h, d)
        off = h * d
    recon = vals[off: off + k * h * d].reshape(k, h, d)
    dist = vals[off + k * h * d: off + k * h * d + k * h].reshape(k, h)
    res = words[:_capi.SF_RESULT_WORDS]
    branch = tuple(int(x) for x in words[_capi.SF_RESULT_WORDS: _capi.SF_RESULT_WORDS + k])
    return draft, recon, dist, branch, res


def _raise_nonfinite(res, taus):
    nf = int(res[_capi.RES_NONFINITE])
    if nf >= 0:
        raise FloatingPointError(f"velocity produced non-finite values at tau={taus[nf]}")


def _report(recon, dist, branch, res, seed) -> VerifierReport:
    return VerifierReport(
        reconstructed=recon.copy(), distances=dist.copy(), branch_prefixes=branch,
        prefix=int(res[_capi.RES_PREFIX]), gripper_switch_detected=bool(res[_capi.RES_SWITCH]),
        shared_noise_seed=seed, decision=_capi.PATH_CODES[int(res[_capi.RES_PATH])],
        planned=int(res[_capi.RES_PLANNED]))


def _check_tiny_inputs(field: VelocityField, draft_net, din, eps, emb, st) -> None:
    """The fused kernel packs its inputs back to back, so every size is checked
    before the launch with the reference's exceptions (flowpolicy.py:253-257
    ``velocity``; nets.py:94-99 ``forward`` for a mis-sized pack or draft
    feature vector)."""
    h, d = field.horizon, field.dim
    if draft_net is None:
        if din.shape != (h, d):
            raise ValueError(f"chunk shape {din.shape} does not match field")
    elif din.size != draft_net.in_dim:
        raise ValueError(f"input has shape {din.shape}, expected ({draft_net.in_dim},)")
    if eps.shape != (h, d):
        raise ValueError("draft and noise shapes differ")
    if emb.size != field.emb_dim or st.size != field.state_dim:
        n = h * d + 1 + emb.size + st.size
        raise ValueError(f"input has shape ({n},), expected ({field.net.in_dim},)")


def tiny_flash_round(field: VelocityField, draft_net, draft_in, cache: ConditioningCache, state,
                     eps, cfg: VerifierConfig, current_sign: float, layout, seed=None,
                     phase_fallback=True, prefix_cap=True, replan_size=12):
    """One fused ``sf_tiny_flash_round`` launch. ``draft_net`` None means
    ``draft_in`` is the draft chunk; otherwise the draft MLP runs on device.
    Returns (draft values, VerifierReport)."""
    h, d = field.horizon, field.dim
    k = len(cfg.timesteps)
    emb = np.asarray(cache.embedding, dtype=np.float64)
    st = np.asarray(state, dtype=np.float64)
    din = np.asarray(draft_in, dtype=np.float64)
    eps = np.asarray(eps, dtype=np.float64)
    _check_tiny_inputs(field, draft_net, din, eps, emb, st)
    n_out = h * d + k * h * d + k * h
    n_words = _capi.SF_RESULT_WORDS + k
    stg = _device.Staging.get("flash", din.size + eps.size + emb.size + st.size + 3, n_out, n_words)
    p_draft, p_eps, p_emb, p_state = stg.upload([din, eps, emb, st])
    out = stg.extra.get("vout")
    if out is None:
        out = stg.extra["vout"] = _capi.SfVerifyOut(
            stg.out_ptr(0), stg.out_ptr(h * d), stg.out_ptr(h * d + k * h * d),
            stg.word_ptr(_capi.SF_RESULT_WORDS), stg.word_ptr(0))
    c = make_cfg(cfg, current_sign, phase_fallback, prefix_cap, replan_size)
    _capi.check(_capi.lib().sf_tiny_flash_round(
        _device.code(), draft_net.device().desc if draft_net is not None else None, p_draft,
        field.net.device().desc, p_emb, field.emb_dim, p_state, field.state_dim, p_eps, h, d,
        layout.continuous_dims, c, out, _device.stream_ptr()), "flash round")
    vals, words = stg.download(n_out, n_words)
    draft, recon, dist, branch, res = _decode(vals, words, k, h, d, seed, True)
    _raise_nonfinite(res, cfg.timesteps)
    return draft, _report(recon, dist, branch, res, seed)


def _run_epilogue(draft, eps, vel, cfg: VerifierConfig, current_sign, cdims, check=True,
                  phase_fallback=True, prefix_cap=True, replan_size=12):
    h, d = draft.shape
    k = vel.shape[0]
    n_out = k * h * d + k * h
    n_words = _capi.SF_RESULT_WORDS + k
    stg = _device.Staging.get("epi", draft.size * 2 + vel.size, n_out, n_words)
    p_draft, p_eps, p_vel = stg.upload([draft, eps, vel])
    out = _capi.SfVerifyOut(None, stg.out_ptr(0), stg.out_ptr(k * h * d),
                            stg.word_ptr(_capi.SF_RESULT_WORDS), stg.word_ptr(0))
    c = make_cfg(cfg, current_sign, phase_fallback, prefix_cap, replan_size)
    _capi.check(_capi.lib().sf_verify_epilogue(_device.code(), p_draft, p_eps, p_vel, h, d, cdims,
                                               c, out, _device.stream_ptr()), "verify epilogue")
    vals, words = stg.download(n_out, n_words)
    _, recon, dist, branch, res = _decode(vals, words, k, h, d, None, False)
    if check:
        _raise_nonfinite(res, cfg.timesteps)
        return recon, dist, branch, res
    return recon.reshape(k, h * d), dist, branch, res


def verify(field, draft: ActionChunk, cache: ConditioningCache, state, cfg: VerifierConfig,
           rng: np.random.Generator, current_gripper_sign: float = -1.0,
           noise_seed: int | None = None) -> VerifierReport:
    """All K branches against one shared noise draw (verifier.py:109-150)."""
    if draft.space != STANDARDIZED:
        raise ValueError("verification operates on standardized drafts")
    if current_gripper_sign not in (-1.0, 1.0):
        raise ValueError("current_sign must be -1.0 or +1.0")
    eps = rng.standard_normal(draft.values.shape)  # one shared draw (verifier.py:129)
    k = len(cfg.timesteps)
    if hasattr(field, "device_verify"):
        field.eval_count += k
        return field.device_verify(draft, cache, state, cfg, eps, current_gripper_sign, noise_seed)
    if isinstance(field, VelocityField) and k <= _capi.TINY_MAX_K:
        field.eval_count += k
        _, rep = tiny_flash_round(field, None, draft.values, cache, state, eps, cfg,
                                  current_gripper_sign, draft.layout, noise_seed)
        return rep
    # generic field protocol (and MLP fields with K > TINY_MAX_K): device
    # interpolation, field evaluated where it lives (branch by branch, as the
    # reference schedules them), device epilogue
    vals = draft.values
    xs = np.empty((k,) + vals.shape)
    da, de = _device.to_dev(vals), _device.to_dev(eps)
    dx = torch.empty(k * vals.size, dtype=da.dtype, device=da.device)
    _capi.check(_capi.lib().sf_interpolate(_device.code(), da.data_ptr(), de.data_ptr(),
                                           _capi.host_doubles(cfg.timesteps), k, vals.size,
                                           dx.data_ptr(), _device.stream_ptr()), "interpolate")
    xs[:] = _device.to_host(dx).reshape(xs.shape)
    vel = np.stack([velocity(field, xs[i], tau, cache, state) for i, tau in enumerate(cfg.timesteps)])
    recon, dist, branch, res = _run_epilogue(vals, eps, vel, cfg, current_gripper_sign,
                                             draft.layout.continuous_dims)
    return _report(recon, dist, branch, res, noise_seed)
