"""Speculative / full rounds and the phase-aware fallback gate.

Mirrors the hot-path half of ``specflow.runtime`` (runtime.py:43-198,
:247-323): ``Models``, ``RuntimePolicy``, ``full_round``, ``flash_attempt``
and the fallback decision. ``flash_attempt`` is ONE device launch for the tiny
models (draft forward + K-branch verify + gate + decision fused); the
decision is evaluated on the device and returned in ``report.decision``.
The conveyor episode loop and latency cost model (runtime.py:201-334,
latency.py) are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np

from .actions import ActionChunk, ChannelLayout, Standardizer, gripper_switch
from .draft import DraftModel, propose
from .flowpolicy import (ConditioningCache, ContextEncoder, DenoiseConfig, VelocityField, denoise,
                         encode_context, _run_full)
from . import _capi
from .actions import STANDARDIZED
from .verifier import VerifierConfig, VerifierReport, tiny_flash_round, verify

MODE_FULL_ONLY = "full_only"
MODE_FLASH = "flash"

PATH_FULL = "full"
PATH_PERIODIC = "periodic_refresh"
PATH_FLASH_ACCEPTED = "flash_accepted"
PATH_FLASH_REJECTED = "flash_rejected_fallback"
PATH_FLASH_PHASE = "flash_phase_fallback"

_DENOISE_STREAM = 0
_VERIFY_STREAM = 1


@dataclass
class Models:
    """Model bundle shared by both paths (runtime.py:43-64)."""

    encoder: ContextEncoder
    field: VelocityField
    standardizer: Standardizer
    draft: DraftModel | None = None

    @property
    def layout(self) -> ChannelLayout:
        assert self.field.layout is not None
        return self.field.layout

    def norm_state(self, robot_state) -> np.ndarray:
        return self.encoder.normalizer.norm_state(robot_state)

    def gripper_sign(self, raw_gripper_state: float) -> float:
        gi = self.layout.gripper_index
        z = (raw_gripper_state - self.standardizer.mean[gi]) / self.standardizer.std[gi]
        return 1.0 if z > 0.0 else -1.0


@dataclass(frozen=True)
class RuntimePolicy:
    """Scheduler knobs (runtime.py:67-88)."""

    mode: str = MODE_FLASH
    replan_size: int = 12
    periodic_refresh: int = 2
    phase_fallback: bool = True
    verifier_cfg: VerifierConfig = dc_field(default_factory=VerifierConfig)
    denoise_cfg: DenoiseConfig = dc_field(default_factory=DenoiseConfig)
    prefix_cap: bool = True
    fallback_accounting: str = "additive"

    def __post_init__(self) -> None:
        if self.mode not in (MODE_FULL_ONLY, MODE_FLASH):
            raise ValueError(f"unknown runtime mode {self.mode!r}")
        if self.replan_size < 1:
            raise ValueError("replan_size must be >= 1")
        if self.periodic_refresh < 0:
            raise ValueError("periodic_refresh must be >= 0")
        if self.fallback_accounting not in ("additive", "full_only"):
            raise ValueError(f"unknown fallback accounting {self.fallback_accounting!r}")


@dataclass
class RunnerState:
    """Between-round scheduler state (runtime.py:133-139)."""

    cache: ConditioningCache | None = None
    flash_since_refresh: int = 0
    gripper_sign: float = -1.0


def detect_gripper_switch(chunks, layout: ChannelLayout, current_sign: float,
                          window: int | None = None) -> bool:
    """runtime.py:142-149."""
    return any(gripper_switch(c, layout, current_sign, window) for c in chunks)


def stream_seed(episode_seed: int, round_index: int, stream: int) -> int:
    """Per-round noise stream seed (runtime.py:152-154)."""
    return int(np.random.SeedSequence([int(episode_seed), int(round_index), int(stream)])
               .generate_state(1)[0])


_stream_seed = stream_seed


def forced_refresh(state: RunnerState, policy: RuntimePolicy) -> bool:
    """Periodic-refresh check made before the attempt (runtime.py:247-250)."""
    return policy.periodic_refresh > 0 and state.flash_since_refresh >= policy.periodic_refresh


def fallback_decision(report: VerifierReport, policy: RuntimePolicy, horizon: int):
    """(path, planned) for a flash attempt (runtime.py:286-320). The device
    computes the same decision in-kernel; this host form serves reports
    produced under a different policy."""
    phase_fb = policy.phase_fallback and report.gripper_switch_detected
    if phase_fb or report.prefix == 0:
        return (PATH_FLASH_PHASE if phase_fb else PATH_FLASH_REJECTED), policy.replan_size
    cap = policy.replan_size if policy.prefix_cap else horizon
    return PATH_FLASH_ACCEPTED, min(report.prefix, cap)


def full_round(obs, models: Models, policy: RuntimePolicy, round_index: int, tick: int,
               episode_seed: int):
    """Context encode + N-step denoise in ONE device launch (runtime.py:157-170)."""
    seed = stream_seed(episode_seed, round_index, _DENOISE_STREAM)
    rng = np.random.default_rng(seed)
    field = models.field
    if isinstance(field, VelocityField):
        feats = models.encoder.features(obs)
        start = rng.standard_normal((field.horizon, field.dim))
        n = policy.denoise_cfg.num_steps
        field.eval_count += n
        vals, emb, st = _run_full(models.encoder.net, feats, models.encoder.embed_dim, field.net,
                                  models.norm_state(obs.robot_state), start, field.horizon,
                                  field.dim, n)
        if st[0] >= 0:
            step = int(st[0])
            if st[1]:
                raise FloatingPointError(f"velocity produced non-finite values at tau={step / n}")
            raise FloatingPointError(f"denoising diverged at step {step} (tau={step / n})")
        cache = ConditioningCache(embedding=emb, captured_round=round_index, captured_tick=tick)
        chunk = ActionChunk(values=vals, layout=field.layout, space=STANDARDIZED)
        return chunk, cache, seed
    cache = encode_context(models.encoder, obs, round_index=round_index, tick=tick)
    chunk = denoise(field, cache, models.norm_state(obs.robot_state), policy.denoise_cfg, rng)
    return chunk, cache, seed


def flash_attempt(obs, models: Models, policy: RuntimePolicy, state: RunnerState,
                  round_index: int, episode_seed: int):
    """Draft from the fresh observation, verify against the stale cache, and
    decide — fused in ONE device launch for the tiny models (runtime.py:173-198)."""
    if state.cache is None:
        raise RuntimeError("flash round requires a cached context from a prior full round")
    if models.draft is None:
        raise RuntimeError("flash mode requires a draft model")
    seed = stream_seed(episode_seed, round_index, _VERIFY_STREAM)
    rng = np.random.default_rng(seed)
    field = models.field
    norm_state = models.norm_state(obs.robot_state)
    if isinstance(field, VelocityField) and len(policy.verifier_cfg.timesteps) <= _capi.TINY_MAX_K:
        draft = models.draft
        feats = draft.features(obs)
        eps = rng.standard_normal((draft.horizon, draft.layout.dim))
        field.eval_count += len(policy.verifier_cfg.timesteps)
        values, report = tiny_flash_round(
            field, draft.net, feats, state.cache, norm_state, eps, policy.verifier_cfg,
            state.gripper_sign, draft.layout, seed, policy.phase_fallback, policy.prefix_cap,
            policy.replan_size)
        chunk = ActionChunk(values=values, layout=draft.layout, space=STANDARDIZED)
        return chunk, report, seed
    chunk = propose(models.draft, obs)
    report = verify(field, chunk, state.cache, norm_state, policy.verifier_cfg, rng,
                    current_gripper_sign=state.gripper_sign, noise_seed=seed)
    return chunk, report, seed
