"""torch restatement of ``oracle/pi0_oracle.py`` — TEST INFRASTRUCTURE ONLY.

The same builder-defined pi0-scale Action Expert, vectorised
over envs x branches so the full cfg3/cfg4 shapes check in seconds. Two
precision modes:

* ``mirror_bf16=True``  — rounds to bf16 at exactly the points
  ``pi0_oracle.field_velocity`` does (the device's storage points); used to
  check DECISIONS (prefixes, switch, path), which must match except rounds
  whose deciding distance lies near delta.
* ``mirror_bf16=False`` — the unrounded fp32 model: same (bf16-valued)
  weights and prefix KV, every activation kept in fp32. This is the north-star
  precision reference: the device's bf16-activation / fp32-accumulate
  endpoints are held to rtol 1e-2 against it (BASELINE.json north_star).

Matmuls run with TF32 disabled (true fp32). Pinned to the numpy oracle by
``tests/test_oracle_torch_cpu.py`` (bitwise init, velocities and drafts at
reduced shapes), which is itself the specification of the model; everything
downstream of the field (interpolate / reconstruct / distances / prefix /
gate / decision) is ``oracle/specflow_oracle.py``, pinned to the reference's
goldens (verifier.py:65-150, actions.py:168-211, runtime.py:286-320).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .pi0_oracle import (TID_A_W, TID_DRAFT_BASE, TID_KV_BASE, TID_LAYER_BASE, TID_OUT_W, TID_S_W,
                         TID_T1_W, TID_T2_W, AEConfig, rope_table, time_features)

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def hash_uniform(seed: int, tid: int, shape, std: float, device="cpu") -> torch.Tensor:
    """pi0_oracle.hash_uniform (splitmix64 counter init) in torch int64
    arithmetic (wrapping multiply, logical shifts): bit-identical float32."""
    n = int(np.prod(shape))
    base = _s64(seed * 0x9E3779B97F4A7C15 + tid * 0xD1B54A32D192ED03)
    z = torch.arange(n, dtype=torch.int64, device=device) + base
    z = (z ^ _lsr(z, 30)) * _s64(0xBF58476D1CE4E5B9)
    z = (z ^ _lsr(z, 27)) * _s64(0x94D049BB133111EB)
    z = z ^ _lsr(z, 31)
    u = _lsr(z, 40).to(torch.float32) * np.float32(2.0 ** -24)
    a = np.float32(std * np.sqrt(3.0))
    return ((u * np.float32(2.0) - np.float32(1.0)) * a).reshape(tuple(shape))


def bf16r(x: torch.Tensor) -> torch.Tensor:
    """Round-to-nearest-even to bf16, kept as float32 (pi0_oracle.bf16)."""
    return x.to(torch.bfloat16).to(torch.float32)


def _gelu_tanh(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


class Pi0Torch:
    """Weights (natural layout, bf16-valued float32), prefix KV of envs
    ``env_ids`` and the field/draft forwards of pi0_oracle in torch."""

    def __init__(self, cfg: AEConfig = AEConfig(), seed: int = 0, kv_seed: int = 1, env_ids=(0,),
                 device="cpu", std: float = 0.02):
        self.cfg, self.device = cfg, device
        W, nq, hd = cfg.width, cfg.q_heads * cfg.head_dim, cfg.head_dim

        def g(tid, *shape):
            return bf16r(hash_uniform(seed, tid, shape, std, device))

        def f32(tid, *shape):
            return hash_uniform(seed, tid, shape, std, device)

        self.a_w, self.s_w = f32(TID_A_W, W, cfg.action_dim), f32(TID_S_W, W, cfg.state_dim)
        self.t1_w, self.t2_w = f32(TID_T1_W, W, W), f32(TID_T2_W, W, W)
        self.out_w = g(TID_OUT_W, cfg.action_dim, W)
        self.layers = []
        for l in range(cfg.layers):
            b = TID_LAYER_BASE + 4 * l
            self.layers.append({"qkv": g(b, nq + 2 * hd, W), "o": g(b + 1, W, nq),
                                "gu": g(b + 2, 2 * cfg.mlp, W), "down": g(b + 3, W, cfg.mlp)})
        # biases are zero in the shared initialiser (pi0_oracle.make_weights)
        self.env_ids = list(env_ids)
        E, P = len(self.env_ids), cfg.prefix_len
        self.kp = torch.empty((cfg.layers, E, P, hd), device=device)
        self.vtp = torch.empty((cfg.layers, E, hd, P), device=device)
        for i, e in enumerate(self.env_ids):
            for l in range(cfg.layers):
                t = TID_KV_BASE + 2 * (e * cfg.layers + l)
                self.kp[l, i] = bf16r(hash_uniform(kv_seed, t, (P, hd), 1.0, device))
                self.vtp[l, i] = bf16r(hash_uniform(kv_seed, t + 1, (hd, P), 1.0, device))
        cs = torch.from_numpy(rope_table(cfg, P + cfg.seg_len)).to(device)
        self.cos, self.sin = cs[..., 0], cs[..., 1]
        self.draft = None
        if cfg.draft_in > 0:
            hid, hdd = cfg.draft_hidden, cfg.horizon * cfg.action_dim
            shapes = ((hid, cfg.draft_in), (hid, hid), (hdd, hid))
            self.draft = [bf16r(hash_uniform(seed, TID_DRAFT_BASE + i, s, float(np.sqrt(1.0 / s[1])),
                                             device)) for i, s in enumerate(shapes)]

    # --------------------------------------------------------------- pieces
    def temb(self, tau: float) -> torch.Tensor:
        f = torch.from_numpy(time_features(self.cfg, tau)).to(self.device, self.t1_w.dtype)
        h = self.t1_w @ f
        h = h / (1.0 + torch.exp(-h))
        return self.t2_w @ h

    @staticmethod
    def _rms(x, eps):
        return 1.0 / torch.sqrt((x * x).sum(-1) / x.shape[-1] + eps)

    def _rope(self, x, pos):
        c, s = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        a, b = x[..., :128], x[..., 128:]
        return torch.cat([a * c - b * s, b * c + a * s], dim=-1)

    @torch.no_grad()
    def velocity(self, x: torch.Tensor, taus, state: torch.Tensor, mirror_bf16: bool = True,
                 env_index=None) -> torch.Tensor:
        """x [E, R, H, D], taus [R], state [E, S] -> v [E, R, H, D] (field
        velocity of branch r at tau_r, attending to env e's prefix KV; env e
        of the batch uses prefix slot env_index[e], default e)."""
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            return self._velocity(x, taus, state, mirror_bf16, env_index)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev

    def _velocity(self, x, taus, state, mirror_bf16, env_index):
        cfg = self.cfg
        rd = bf16r if mirror_bf16 else (lambda t: t)
        E, R, H, D = x.shape
        T, P, W = cfg.seg_len, cfg.prefix_len, cfg.width
        nq, hd, nh = cfg.q_heads * cfg.head_dim, cfg.head_dim, cfg.q_heads
        dt = self.a_w.dtype
        x = x.to(self.device, dt)
        state = state.to(self.device, dt)
        env_index = list(range(E)) if env_index is None else list(env_index)
        temb = torch.stack([self.temb(float(t)) for t in taus])             # [R, W]
        h = torch.empty((E, R, T, W), device=self.device, dtype=dt)
        h[:, :, 0] = (state @ self.s_w.T)[:, None, :]
        h[:, :, 1:] = x @ self.a_w.T + temb[None, :, None, :]
        h = h.reshape(E * R * T, W)
        pos = P + torch.arange(T, device=self.device)
        posr = pos.repeat(E * R)
        scale = 1.0 / math.sqrt(hd)
        # state token (t = 0) sees the prefix and itself; action tokens the whole segment
        smask = torch.ones((T, T), dtype=torch.bool, device=self.device)
        smask[0, 1:] = False
        for l, Lw in enumerate(self.layers):
            r = self._rms(h, cfg.eps)
            qkv = (rd(h) @ Lw["qkv"].T) * r[:, None]
            q = rd(self._rope(qkv[:, :nq].reshape(-1, nh, hd), posr)).reshape(E, R, T, nh, hd)
            k = rd(self._rope(qkv[:, nq:nq + hd].reshape(-1, 1, hd), posr)).reshape(E, R, T, hd)
            v = rd(qkv[:, nq + hd:]).reshape(E, R, T, hd)
            o = torch.empty((E, R, T, nh, hd), device=self.device, dtype=dt)
            for e in range(E):
                kp = self.kp[l, env_index[e]]                                # [P, hd]
                vp = self.vtp[l, env_index[e]].T                             # [P, hd]
                sp = torch.einsum("rthd,pd->rthp", q[e], kp)
                ss = torch.einsum("rthd,rsd->rths", q[e], k[e])
                ss = ss.masked_fill(~smask[None, :, None, :], float("-inf"))
                s = torch.cat([sp, ss], dim=-1) * scale                      # [R, T, nh, P+T]
                m = s.amax(-1, keepdim=True)
                p = torch.exp(s - m)
                lsum = p.sum(-1, keepdim=True)
                pr = rd(p)
                oe = torch.einsum("rthp,pd->rthd", pr[..., :P], vp) + \
                    torch.einsum("rths,rsd->rthd", pr[..., P:], v[e])
                o[e] = oe / lsum
            o = rd(o.reshape(-1, nq))
            h = h + o @ Lw["o"].T
            r2 = self._rms(h, cfg.eps)
            gu = (rd(h) @ Lw["gu"].T) * r2[:, None]
            hh = rd(_gelu_tanh(gu[:, :cfg.mlp]) * gu[:, cfg.mlp:])
            h = h + hh @ Lw["down"].T
        h = h.reshape(E, R, T, W)
        rf = self._rms(h[:, :, 1:], cfg.eps)
        return (rd(h[:, :, 1:]) @ self.out_w.T) * rf[..., None]

    @torch.no_grad()
    def draft_forward(self, obs: torch.Tensor, mirror_bf16: bool = True,
                      gripper_bias: float = 0.0) -> torch.Tensor:
        """pi0_oracle.draft_forward: bf16 operands, fp32 accumulation, bf16
        hidden activations (obs [B, F] -> [B, H, D]); ``gripper_bias`` is the
        output bias of the gripper column (ActionExpert draft_gripper_bias)."""
        rd = bf16r if mirror_bf16 else (lambda t: t)
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            a = rd(obs.to(self.device, torch.float32))
            for i, w in enumerate(self.draft):
                z = a @ w.T
                a = rd(torch.tanh(z)) if i < 2 else z
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        a = a.reshape(-1, self.cfg.horizon, self.cfg.action_dim)
        if gripper_bias:
            a[:, :, -1] += gripper_bias
        return a
