"""numpy restatement of the pi0-scale Action Expert field — TEST INFRASTRUCTURE ONLY.

No reference implementation of this model exists: the reference package
substitutes MLPs and BASELINE configs 3-4 ask for "a pi0-scale
Action Expert (~300M, 18 layers, width 1024) over a random-init 2B-VLM prefix
KV cache". The architecture below is the builder's definition,
written to the paper's description (PAPER.md:81-96, :131 block mask) and
gemma_300m-style dimensions; this file IS its specification. Everything
downstream of the field (interpolation, reconstruction, distances, prefix,
gate, decision, Euler) is the reference's and is checked with
``oracle/specflow_oracle.py``, which is pinned to the reference's goldens.

Precision model (identical rounding points to the device path):
  * weights are bf16; GEMM operands are bf16; accumulation fp32;
  * the residual stream x is fp32; an RMSNorm feeding a GEMM is applied to the
    fp32 accumulator (r[m] * (bf16(x) @ W^T)), eps = 1e-6;
  * q, k (after RoPE), v, softmax P, attention output and GeGLU output are
    rounded to bf16 where the device stores them;
  * the action head output (velocity) is fp32.
``field_velocity(..., bf16_points=False)`` is the unrounded fp32 model (same
bf16-valued weights and KV, activations never rounded): the north star's
precision reference and the fp32 mode's (SF_AE_FP32) target.
Parity is "unpinned" against any external reference for this model (there is
none); GPU parity is checked against this oracle at reduced depth/width and,
through its torch port (oracle/pi0_torch.py), at full cfg3/cfg4 size.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def bf16(a):
    """Round-to-nearest-even to bfloat16, returned as float32."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    r = ((u + rounding) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(a), a, out)


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
    draft_in: int = 64
    draft_hidden: int = 1024

    @property
    def seg_len(self) -> int:
        return 1 + self.horizon


def rope_table(cfg: AEConfig, max_pos: int) -> np.ndarray:
    """(cos, sin) [max_pos, head_dim/2] as float32 (rotate_half convention)."""
    half = cfg.head_dim // 2
    inv = cfg.rope_base ** (-np.arange(half, dtype=np.float64) * 2.0 / cfg.head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)


def time_features(cfg: AEConfig, tau: float) -> np.ndarray:
    """sin/cos time features (float64 -> float32), pi0-style periods."""
    half = cfg.width // 2
    frac = np.linspace(0.0, 1.0, half)
    period = cfg.temb_min_period * (cfg.temb_max_period / cfg.temb_min_period) ** frac
    ang = 2.0 * np.pi * tau / period
    return np.concatenate([np.sin(ang), np.cos(ang)]).astype(np.float32)


def time_embedding(cfg, w, tau):
    """temb(tau) = W_t2 swish(W_t1 f + b_t1) + b_t2 (fp32 weights, fp32 math)."""
    f = time_features(cfg, tau)
    h = w["t1_w"] @ f + w["t1_b"]
    h = h / (1.0 + np.exp(-h))
    return (w["t2_w"] @ h + w["t2_b"]).astype(np.float32)


def _rms(x, eps):
    return 1.0 / np.sqrt((x.astype(np.float32) ** 2).sum(-1, dtype=np.float32) / x.shape[-1] + eps)


def _mm(a_bf16, w_bf16):
    return (a_bf16.astype(np.float32) @ w_bf16.astype(np.float32).T).astype(np.float32)


def _rope(x, cs, pos):
    """x [T, heads, 256] with rotate_half pairs (i, i+128) at positions pos [T]."""
    c = cs[pos, :, 0][:, None, :]
    s = cs[pos, :, 1][:, None, :]
    a, b = x[..., :128], x[..., 128:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1).astype(np.float32)


def gelu_tanh(x):
    return (0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))).astype(np.float32)


def embed_tokens(cfg, w, actions, tau, state):
    """One branch: token 0 = state_proj(s), tokens 1..H = action_in(a_h) + temb(tau)."""
    temb = time_embedding(cfg, w, tau)
    x = np.empty((cfg.seg_len, cfg.width), np.float32)
    x[0] = w["s_w"] @ state.astype(np.float32) + w["s_b"]
    x[1:] = actions.astype(np.float32) @ w["a_w"].T + w["a_b"] + temb
    return x


def field_velocity(cfg, w, kv, branches, state, bf16_points=True):
    """Velocity for several branches that share the prefix KV.

    branches: list of (actions [H, D], tau); kv: (K [L][P, 256], Vt [L][256, P])
    bf16-valued float32 arrays. Returns v [len(branches), H, D] float32.
    bf16_points=False is the unrounded fp32 model: same (bf16-valued) weights
    and prefix KV, activations never rounded (the north-star fp32 reference).
    """
    bf16 = globals()["bf16"] if bf16_points else (lambda a: np.asarray(a, np.float32))
    cs = rope_table(cfg, cfg.prefix_len + cfg.seg_len)
    kp, vtp = kv
    P = cfg.prefix_len
    T = cfg.seg_len
    xs = [embed_tokens(cfg, w, a, t, state) for a, t in branches]
    pos = P + np.arange(T)
    scale = 1.0 / np.sqrt(cfg.head_dim)
    out = []
    for x in xs:
        for l in range(cfg.layers):
            L = w["layers"][l]
            r = _rms(x, cfg.eps)
            xb = bf16(x)
            qkv = _mm(xb, L["qkv"]) * r[:, None]
            nq = cfg.q_heads * cfg.head_dim
            q = qkv[:, :nq].reshape(T, cfg.q_heads, cfg.head_dim)
            k = qkv[:, nq: nq + cfg.head_dim].reshape(T, 1, cfg.head_dim)
            v = bf16(qkv[:, nq + cfg.head_dim:])
            q = bf16(_rope(q, cs, pos))
            k = bf16(_rope(k, cs, pos))[:, 0]
            keys = np.concatenate([kp[l], k], 0)          # [P+T, 256]
            vals = np.concatenate([vtp[l].T, v], 0)       # [P+T, 256]
            s = np.einsum("thd,kd->thk", q, keys).astype(np.float32) * scale
            mask = np.ones((T, P + T), bool)
            mask[0, P + 1:] = False                        # state token: prefix + itself
            s = np.where(mask[:, None, :], s, -np.inf)
            m = s.max(-1, keepdims=True)
            p = np.exp(s - m)
            lsum = p.sum(-1, keepdims=True)
            o = np.einsum("thk,kd->thd", bf16(p), vals).astype(np.float32) / lsum
            o = bf16(o.reshape(T, nq))
            x = x + _mm(o, L["o"])
            r2 = _rms(x, cfg.eps)
            gu = _mm(bf16(x), L["gu"]) * r2[:, None]
            h = bf16(gelu_tanh(gu[:, : cfg.mlp]) * gu[:, cfg.mlp:])
            x = x + _mm(h, L["down"])
        rf = _rms(x, cfg.eps)
        v = _mm(bf16(x[1:]), w["out_w"]) * rf[1:, None] + w["out_b"]
        out.append(v.astype(np.float32))
    return np.stack(out)


_M64 = (1 << 64) - 1


def hash_uniform(seed: int, tid: int, shape, std: float) -> np.ndarray:
    """Counter-based init shared bit-for-bit with the device initialiser
    (csrc/pi0.cu ``fill_hash_uniform``): splitmix64 of (seed, tensor id,
    flat index) -> 24 uniform bits -> (2u - 1) * std * sqrt(3) in float32."""
    n = int(np.prod(shape))
    with np.errstate(over="ignore"):
        z = (np.uint64((seed * 0x9E3779B97F4A7C15 + tid * 0xD1B54A32D192ED03) & _M64)
             + np.arange(n, dtype=np.uint64))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    a = np.float32(std * np.sqrt(3.0))
    return ((u * np.float32(2.0) - np.float32(1.0)) * a).astype(np.float32).reshape(shape)


# tensor ids for hash_uniform (device init uses the same table)
TID_A_W, TID_S_W, TID_T1_W, TID_T2_W, TID_OUT_W = 1, 2, 3, 4, 5
TID_DRAFT_BASE = 20   # + {0, 1, 2}: draft MLP layers
TID_LAYER_BASE = 100  # + 4 * layer + {0: qkv, 1: o, 2: gu, 3: down}


def make_draft_weights(cfg: AEConfig, seed: int = 0):
    """tanh MLP draft [draft_in -> hid -> hid -> H*D], bf16 weights with std
    sqrt(1/fan_in), zero fp32 biases (draft.py:29-61 at pi0 scale)."""
    hid, hd = cfg.draft_hidden, cfg.horizon * cfg.action_dim
    shapes = ((hid, cfg.draft_in), (hid, hid), (hd, hid))
    ws = [bf16(hash_uniform(seed, TID_DRAFT_BASE + i, s, float(np.sqrt(1.0 / s[1]))))
          for i, s in enumerate(shapes)]
    return ws, [np.zeros(s[0], np.float32) for s in shapes]


def draft_forward(cfg: AEConfig, dw, obs):
    """propose(): bf16 operands, fp32 accumulation, bf16 hidden activations."""
    ws, bs = dw
    a = bf16(obs)
    for i, (w, b) in enumerate(zip(ws, bs)):
        z = _mm(a, w) + b
        a = bf16(np.tanh(z)) if i < 2 else z.astype(np.float32)
    return a.reshape(-1, cfg.horizon, cfg.action_dim)
TID_KV_BASE = 10000   # + 2 * (env * layers + layer) + {0: K, 1: V^T}


def make_weights(cfg: AEConfig, seed: int = 0, std: float = 0.02):
    """Weights in the NATURAL layout (bf16-valued float32 except the fp32
    embedding/time MLP and head bias). The device builds the same values in
    its interleaved layouts."""

    def g(tid, *shape):
        return bf16(hash_uniform(seed, tid, shape, std))

    W, nq = cfg.width, cfg.q_heads * cfg.head_dim
    w = {
        "a_w": hash_uniform(seed, TID_A_W, (W, cfg.action_dim), std), "a_b": np.zeros(W, np.float32),
        "s_w": hash_uniform(seed, TID_S_W, (W, cfg.state_dim), std), "s_b": np.zeros(W, np.float32),
        "t1_w": hash_uniform(seed, TID_T1_W, (W, W), std), "t1_b": np.zeros(W, np.float32),
        "t2_w": hash_uniform(seed, TID_T2_W, (W, W), std), "t2_b": np.zeros(W, np.float32),
        "out_w": g(TID_OUT_W, cfg.action_dim, W), "out_b": np.zeros(cfg.action_dim, np.float32),
        "layers": [],
    }
    for l in range(cfg.layers):
        b = TID_LAYER_BASE + 4 * l
        w["layers"].append({
            "qkv": g(b + 0, nq + 2 * cfg.head_dim, W),
            "o": g(b + 1, W, nq),
            "gu": g(b + 2, 2 * cfg.mlp, W),   # rows [0, mlp) gate, [mlp, 2 mlp) up
            "down": g(b + 3, W, cfg.mlp),
        })
    return w


def make_prefix_kv(cfg: AEConfig, seed: int = 1, env: int = 0):
    """Random prefix KV of one env (unit std): K [L][P, 256], V^T [L][256, P]."""
    kp, vtp = [], []
    for l in range(cfg.layers):
        t = TID_KV_BASE + 2 * (env * cfg.layers + l)
        kp.append(bf16(hash_uniform(seed, t, (cfg.prefix_len, cfg.head_dim), 1.0)))
        vtp.append(bf16(hash_uniform(seed, t + 1, (cfg.head_dim, cfg.prefix_len), 1.0)))
    return kp, vtp


# ---------------------------------------------------------------- VLM prefill
# Context refresh: the prefix encoder whose per-layer K / V
# form the Action Expert's prefix KV pool. Builder-defined (the reference's
# encode_context, flowpolicy.py:156-161, is a tiny MLP; the paper's prefix is
# the Gemma-2B VLM): a decoder stack with bidirectional prefix
# attention, same block structure and numerics conventions as the Action
# Expert above.

TID_VLM_BASE = 1000  # + 4 * layer + {0: qkv, 1: o, 2: gu, 3: down}


@dataclass(frozen=True)
class VLMConfig:
    width: int = 2048
    layers: int = 18
    q_heads: int = 8
    head_dim: int = 256
    mlp: int = 16384
    prefix_len: int = 800
    eps: float = 1e-6
    rope_base: float = 10000.0


def make_vlm_weights(cfg: VLMConfig, seed: int = 7, std: float = 0.02):
    def g(tid, *shape):
        return bf16(hash_uniform(seed, tid, shape, std))

    W, nq = cfg.width, cfg.q_heads * cfg.head_dim
    out = []
    for l in range(cfg.layers):
        b = TID_VLM_BASE + 4 * l
        out.append({"qkv": g(b + 0, nq + 2 * cfg.head_dim, W), "o": g(b + 1, W, nq),
                    "gu": g(b + 2, 2 * cfg.mlp, W), "down": g(b + 3, W, cfg.mlp)})
    return out


def prefill_kv(cfg: VLMConfig, layers, x):
    """One env: token embeddings x [P, W] -> per-layer K [L][P, 256] and
    V^T [L][256, P] (bf16-valued float32), bidirectional attention over the
    P prefix tokens at RoPE positions 0..P-1."""
    P = cfg.prefix_len
    cs = rope_table(cfg, P)
    pos = np.arange(P)
    scale = 1.0 / np.sqrt(cfg.head_dim)
    nq = cfg.q_heads * cfg.head_dim
    x = x.astype(np.float32).copy()
    ks, vts = [], []
    for L in layers:
        r = _rms(x, cfg.eps)
        qkv = _mm(bf16(x), L["qkv"]) * r[:, None]
        q = qkv[:, :nq].reshape(P, cfg.q_heads, cfg.head_dim)
        k = qkv[:, nq: nq + cfg.head_dim].reshape(P, 1, cfg.head_dim)
        v = bf16(qkv[:, nq + cfg.head_dim:])
        q = bf16(_rope(q, cs, pos))
        k = bf16(_rope(k, cs, pos))[:, 0]
        ks.append(k)
        vts.append(np.ascontiguousarray(v.T))
        s = np.einsum("thd,kd->thk", q, k).astype(np.float32) * scale
        m = s.max(-1, keepdims=True)
        p = np.exp(s - m)
        lsum = p.sum(-1, keepdims=True)
        o = np.einsum("thk,kd->thd", bf16(p), v).astype(np.float32) / lsum
        x = x + _mm(bf16(o.reshape(P, nq)), L["o"])
        r2 = _rms(x, cfg.eps)
        gu = _mm(bf16(x), L["gu"]) * r2[:, None]
        h = bf16(gelu_tanh(gu[:, : cfg.mlp]) * gu[:, cfg.mlp:])
        x = x + _mm(h, L["down"])
    return np.stack(ks), np.stack(vts)
