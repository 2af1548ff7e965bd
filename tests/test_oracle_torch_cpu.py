"""Pin the vectorised torch oracle (oracle/pi0_torch.py) to the numpy oracle
(oracle/pi0_oracle.py) on the CPU: bitwise init, velocities and drafts at
reduced shapes. The torch oracle is what the full-size cfg3/cfg4 GPU parity
tests use as their checker."""

import numpy as np
import pytest

SMALL = dict(width=512, layers=2, q_heads=8, head_dim=256, mlp=1024, action_dim=8, state_dim=8,
             horizon=10, prefix_len=64, draft_in=64, draft_hidden=128)


def test_hash_uniform_bitwise():
    import torch

    from oracle import pi0_oracle as po
    from oracle import pi0_torch as pt

    for seed, tid, shape, std in ((0, 1, (37, 129), 0.02), (5, 10123, (3, 1000), 1.0),
                                  (2 ** 40 + 3, 123456, (7,), 0.5)):
        want = po.hash_uniform(seed, tid, shape, std)
        got = pt.hash_uniform(seed, tid, shape, std).numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    x = torch.randn(1000) * 7
    assert np.array_equal(pt.bf16r(x).numpy(), po.bf16(x.numpy()))


@pytest.mark.parametrize("mirror", [True, False])
def test_velocity_matches_numpy_oracle(mirror):
    """Unrounded (fp32) mode: same math, only the fp32 accumulation order
    differs -> agreement at fp32 level. bf16-mirroring mode: identical rounding
    points, but a 1e-7 accumulation-order difference occasionally flips one
    bf16 rounding (an ulp, 2^-8 relative) and the flip propagates through
    softmax / the residual stream, so two fp32 orders agree only to ~1e-3 of
    the velocity norm -- the intrinsic noise floor of any bf16-activation
    implementation, device included (measured: 1.2e-3 after one layer)."""
    import torch

    from oracle import pi0_oracle as po
    from oracle import pi0_torch as pt

    cfg = po.AEConfig(**SMALL)
    E, R = 2, 3
    m = pt.Pi0Torch(cfg, seed=0, kv_seed=1, env_ids=(0, 5))
    w = po.make_weights(cfg, 0)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((E, R, cfg.horizon, cfg.action_dim)).astype(np.float32)
    st = rng.standard_normal((E, cfg.state_dim)).astype(np.float32)
    taus = (0.2, 0.5, 0.8)
    got = m.velocity(torch.from_numpy(x), taus, torch.from_numpy(st), mirror_bf16=mirror).numpy()
    for i, e in enumerate((0, 5)):
        kv = po.make_prefix_kv(cfg, 1, e)
        want = po.field_velocity(cfg, w, kv, [(x[i, r], taus[r]) for r in range(R)], st[i],
                                 bf16_points=mirror)
        if mirror:
            assert np.linalg.norm(got[i] - want) <= 1e-2 * np.linalg.norm(want)
        else:
            np.testing.assert_allclose(got[i], want, rtol=1e-4, atol=1e-5 * np.abs(want).max())


def test_unrounded_mode_is_fp32():
    """mirror_bf16=False keeps activations in fp32: it must differ from the
    mirrored model, and agree with a float64 evaluation far tighter than bf16."""
    import torch

    from oracle import pi0_oracle as po
    from oracle import pi0_torch as pt

    cfg = po.AEConfig(**dict(SMALL, layers=1))
    m = pt.Pi0Torch(cfg, env_ids=(0,))
    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.standard_normal((1, 2, cfg.horizon, cfg.action_dim)).astype(np.float32))
    st = torch.from_numpy(rng.standard_normal((1, cfg.state_dim)).astype(np.float32))
    a = m.velocity(x, (0.3, 0.7), st, mirror_bf16=False)
    b = m.velocity(x, (0.3, 0.7), st, mirror_bf16=True)
    assert not torch.equal(a, b)
    m64 = pt.Pi0Torch(cfg, env_ids=(0,))
    for name in ("a_w", "s_w", "t1_w", "t2_w", "out_w", "kp", "vtp", "cos", "sin"):
        setattr(m64, name, getattr(m64, name).double())
    m64.layers = [{k: v.double() for k, v in L.items()} for L in m64.layers]
    c = m64._velocity(x.double(), (0.3, 0.7), st.double(), False, None)
    np.testing.assert_allclose(a.numpy(), c.numpy(), rtol=1e-4, atol=1e-5 * c.abs().max().item())


def test_draft_matches_numpy_oracle():
    import torch

    from oracle import pi0_oracle as po
    from oracle import pi0_torch as pt

    cfg = po.AEConfig(**SMALL)
    m = pt.Pi0Torch(cfg, env_ids=(0,))
    obs = np.random.default_rng(2).standard_normal((3, cfg.draft_in)).astype(np.float32)
    want = po.draft_forward(cfg, po.make_draft_weights(cfg, 0), obs)
    got = m.draft_forward(torch.from_numpy(obs)).numpy()
    np.testing.assert_allclose(got, want, rtol=2e-3, atol=2e-3 * np.abs(want).max())
