"""Main policy: context encoder, velocity fields, and the device Euler full path.

Mirrors ``specflow.flowpolicy`` (flowpolicy.py:1-306). The hot-path entry
points — ``encode_context``, ``velocity``, ``integrate_flow`` and ``denoise`` —
run on the device:

* the reference's MLP ``VelocityField`` uses the fused tiny kernels
  (``sf_tiny_full_round``: encode + all N Euler steps in one cluster launch;
  ``sf_tiny_field_eval`` for single evaluations);
* the pi0-scale Action Expert (``paper_2605_13778_b200.pi0``) plugs in through
  the same field protocol and runs its own CUDA-graph Euler loop;
* any other object honouring the field protocol (``AnalyticField`` and the
  reference tests' closed-form fields) is evaluated where it lives, with the
  Euler update and finite checks on the device (``sf_euler_update``).

Training (ObsNormalizer.fit / fit_flow_field / train_flow) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _capi, _device
from .actions import STANDARDIZED, ActionChunk, ChannelLayout
from .nets import Mlp


@dataclass(frozen=True)
class Observation:
    """World features, task id and robot state (flowpolicy.py:21-35)."""

    world_features: np.ndarray
    task_id: int
    robot_state: np.ndarray

    def __post_init__(self) -> None:
        wf = np.asarray(self.world_features, dtype=np.float64)
        rs = np.asarray(self.robot_state, dtype=np.float64)
        if not (np.isfinite(wf).all() and np.isfinite(rs).all()):
            raise ValueError("observation contains non-finite entries")
        object.__setattr__(self, "world_features", wf)
        object.__setattr__(self, "robot_state", rs)


@dataclass(frozen=True)
class ConditioningCache:
    """Context snapshot from the last full round (flowpolicy.py:38-50). For the
    pi0-scale expert ``embedding`` is empty and ``kv`` holds the device prefix
    KV cache (the VLM prefill output)."""

    embedding: np.ndarray
    captured_round: int = 0
    captured_tick: int = 0
    kv: object = None

    def __post_init__(self) -> None:
        emb = np.asarray(self.embedding, dtype=np.float64)
        if not np.isfinite(emb).all():
            raise ValueError("cache embedding is non-finite")
        object.__setattr__(self, "embedding", emb)


@dataclass(frozen=True)
class ObsNormalizer:
    """Observation feature scaling (flowpolicy.py:53-114); fitting is training."""

    world_mean: np.ndarray
    world_std: np.ndarray
    state_mean: np.ndarray
    state_std: np.ndarray

    @classmethod
    def identity(cls, world_dim: int, state_dim: int) -> "ObsNormalizer":
        return cls(np.zeros(world_dim), np.ones(world_dim), np.zeros(state_dim), np.ones(state_dim))

    def norm_world(self, world) -> np.ndarray:
        return (np.asarray(world, dtype=np.float64) - self.world_mean) / self.world_std

    def norm_state(self, state) -> np.ndarray:
        return (np.asarray(state, dtype=np.float64) - self.state_mean) / self.state_std


@dataclass
class ContextEncoder:
    """(world features, task id) -> embedding [features, MLP(features)] (flowpolicy.py:117-147)."""

    net: Mlp
    n_tasks: int
    normalizer: ObsNormalizer

    @property
    def embed_dim(self) -> int:
        return self.net.in_dim + self.net.out_dim

    def features(self, obs: Observation) -> np.ndarray:
        if not 0 <= obs.task_id < self.n_tasks:
            raise ValueError(f"unknown task id {obs.task_id}")
        onehot = np.zeros(self.n_tasks)
        onehot[obs.task_id] = 1.0
        return np.concatenate([self.normalizer.norm_world(obs.world_features), onehot])


def _run_full(encoder_net, enc_in, emb_dim, field_net, state, start, horizon, dim, n):
    """One ``sf_tiny_full_round`` launch; returns (chunk, emb, status) on host.
    Inputs go up in one pinned copy, chunk + embedding + status come back in
    one copy (``_device.Staging``)."""
    enc_in = np.asarray(enc_in, dtype=np.float64).ravel()
    st_in = np.asarray(state, dtype=np.float64).ravel()
    start = np.asarray(start, dtype=np.float64).ravel()
    hd = horizon * dim
    ne = max(emb_dim, 1)
    stg = _device.Staging.get("full", enc_in.size + max(st_in.size, 1) + start.size, hd + ne, 2)
    p_in, p_state, p_start = stg.upload([enc_in, st_in if st_in.size else np.zeros(1), start])
    enc_desc = encoder_net.device().desc if encoder_net is not None else None
    field_desc = field_net.device().desc if field_net is not None else None
    _capi.check(_capi.lib().sf_tiny_full_round(
        _device.code(), enc_desc, p_in, emb_dim, field_desc, p_state, int(st_in.size), p_start, horizon,
        dim, n, stg.out_ptr(0), stg.out_ptr(hd), stg.word_ptr(0), _device.stream_ptr()), "full round")
    vals, st = stg.download(hd + ne, 2)
    return vals[:hd].reshape(horizon, dim), vals[hd:hd + emb_dim], st


def encode_context(encoder: ContextEncoder, obs: Observation, round_index: int = 0,
                   tick: int = 0) -> ConditioningCache:
    """Deterministic embedding; robot state excluded (flowpolicy.py:156-161).
    Runs the encoder MLP on device (``sf_tiny_full_round`` with N=0)."""
    feats = encoder.features(obs)
    _, emb, _ = _run_full(encoder.net, feats, encoder.embed_dim, None, np.zeros(0), np.zeros(1), 1,
                          1, 0)
    return ConditioningCache(embedding=emb, captured_round=round_index, captured_tick=tick)


@dataclass
class VelocityField:
    """Endpoint-parameterised MLP field over flattened H x D chunks
    (flowpolicy.py:164-209): v = (net([x, tau, emb, state]) - x) / (1 - tau)."""

    net: Mlp
    horizon: int
    dim: int
    emb_dim: int
    state_dim: int
    layout: ChannelLayout | None = None
    eval_count: int = 0

    def __post_init__(self) -> None:
        want_in = self.horizon * self.dim + 1 + self.emb_dim + self.state_dim
        if self.net.in_dim != want_in or self.net.out_dim != self.horizon * self.dim:
            raise ValueError("velocity net dimensions do not match (H, D, emb, state)")
        if self.layout is not None and self.layout.dim != self.dim:
            raise ValueError("layout does not match chunk dim")

    def evaluate(self, values, tau: float, cache: ConditioningCache, state) -> np.ndarray:
        """One device evaluation (``sf_tiny_field_eval``)."""
        self.eval_count += 1
        v = _field_eval(self, np.asarray(values, dtype=np.float64)[None], [float(tau)], cache, state)
        return v[0]


def _field_eval(field: VelocityField, xs: np.ndarray, taus, cache, state) -> np.ndarray:
    rows = xs.shape[0]
    d_x = _device.to_dev(xs.reshape(rows, -1))
    d_emb = _device.to_dev(cache.embedding if cache.embedding.size else np.zeros(1))
    st = np.asarray(state, dtype=np.float64)
    d_state = _device.to_dev(st if st.size else np.zeros(1))
    out = torch.empty_like(d_x)
    taus_c = _capi.host_doubles(taus)
    _capi.check(_capi.lib().sf_tiny_field_eval(
        _device.code(), field.net.device().desc, d_x.data_ptr(), taus_c, rows, d_emb.data_ptr(),
        field.emb_dim, d_state.data_ptr(), field.state_dim, field.horizon, field.dim,
        out.data_ptr(), None, _device.stream_ptr()), "field evaluation")
    return _device.to_host(out).reshape(rows, field.horizon, field.dim)


@dataclass
class AnalyticField:
    """Closed-form field for self-tests and oracles (flowpolicy.py:212-227)."""

    fn: object
    horizon: int
    dim: int
    layout: ChannelLayout | None = None
    eval_count: int = 0

    def evaluate(self, values, tau: float, cache: ConditioningCache, state) -> np.ndarray:
        self.eval_count += 1
        out = np.asarray(self.fn(np.asarray(values, dtype=np.float64), tau), dtype=np.float64)
        return out.reshape(self.horizon, self.dim)


def straight_line_field(target, layout: ChannelLayout | None = None) -> AnalyticField:
    """v(A, tau) = (target - A) / (1 - tau) (flowpolicy.py:230-239)."""
    goal = np.asarray(target, dtype=np.float64)
    return AnalyticField(fn=lambda v, t: (goal - v) / (1.0 - t), horizon=goal.shape[0],
                         dim=goal.shape[1], layout=layout)


def constant_field(velocity_value, layout: ChannelLayout | None = None) -> AnalyticField:
    vel = np.asarray(velocity_value, dtype=np.float64)
    return AnalyticField(fn=lambda v, t: vel, horizon=vel.shape[0], dim=vel.shape[1], layout=layout)


def velocity(field, values, tau: float, cache: ConditioningCache, state) -> np.ndarray:
    """One checked evaluation (flowpolicy.py:249-261)."""
    if not 0.0 <= tau <= 1.0:
        raise ValueError(f"tau={tau} outside [0, 1]")
    vals = np.asarray(values, dtype=np.float64)
    if vals.shape != (field.horizon, field.dim):
        raise ValueError(f"chunk shape {vals.shape} does not match field")
    out = field.evaluate(vals, tau, cache, state)
    if not np.isfinite(out).all():
        raise FloatingPointError(f"velocity produced non-finite values at tau={tau}")
    return out


@dataclass(frozen=True)
class DenoiseConfig:
    num_steps: int = 10

    def __post_init__(self) -> None:
        if self.num_steps < 1:
            raise ValueError("num_steps must be >= 1")


def integrate_flow(field, cache: ConditioningCache, state, cfg: DenoiseConfig,
                   rng: np.random.Generator) -> np.ndarray:
    """Forward Euler from A^0 ~ N(0, I) on tau_i = i/N (flowpolicy.py:273-292).

    The noise is drawn on the host from the caller's generator exactly as the
    reference does (one ``standard_normal((H, D))`` call), then the whole loop
    runs on the device.
    """
    n = cfg.num_steps
    start = rng.standard_normal((field.horizon, field.dim))
    if hasattr(field, "device_denoise"):
        return field.device_denoise(cache, state, start, n)
    if isinstance(field, VelocityField):
        emb = np.asarray(cache.embedding, np.float64)
        st_in = np.asarray(state, np.float64)
        if emb.size != field.emb_dim or st_in.size != field.state_dim:
            # the reference's nets.forward rejects the mis-sized pack (nets.py:94-99)
            n_in = field.horizon * field.dim + 1 + emb.size + st_in.size
            raise ValueError(f"input has shape ({n_in},), expected ({field.net.in_dim},)")
        field.eval_count += n
        out, _, st = _run_full(None, cache.embedding if cache.embedding.size else np.zeros(0),
                               field.emb_dim, field.net, np.asarray(state, np.float64), start,
                               field.horizon, field.dim, n)
        if st[0] >= 0:
            step = int(st[0])
            if st[1]:
                raise FloatingPointError(f"velocity produced non-finite values at tau={step / n}")
            raise FloatingPointError(f"denoising diverged at step {step} (tau={step / n})")
        return out
    return _generic_integrate(field, cache, state, start, n)


def _generic_integrate(field, cache, state, start, n):
    """Field evaluated by its own protocol; update + finite check on device."""
    lib = _capi.lib()
    d_vals = _device.to_dev(start)
    status = torch.full((1,), -1, dtype=torch.int32, device=d_vals.device)
    for i in range(n):
        tau = i / n
        cur = _device.to_host(d_vals).reshape(start.shape)
        v = velocity(field, cur, tau, cache, state)
        d_v = _device.to_dev(v)
        _capi.check(lib.sf_euler_update(_device.code(), d_vals.data_ptr(), d_v.data_ptr(),
                                        d_vals.numel(), n, i, status.data_ptr(),
                                        _device.stream_ptr()), "euler update")
        if int(status.item()) >= 0:
            raise FloatingPointError(f"denoising diverged at step {i} (tau={tau})")
    return _device.to_host(d_vals).reshape(start.shape)


def denoise(field, cache: ConditioningCache, state, cfg: DenoiseConfig,
            rng: np.random.Generator) -> ActionChunk:
    """integrate_flow wrapped as a standardized chunk (flowpolicy.py:295-306)."""
    if field.layout is None:
        raise ValueError("field has no channel layout; use integrate_flow instead")
    return ActionChunk(values=integrate_flow(field, cache, state, cfg, rng), layout=field.layout,
                       space=STANDARDIZED)
