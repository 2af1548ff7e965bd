"""cfg5-shaped parity of the tiny path (K in {1, 2, 4, 8},
H in {16, 50, 100}) against the pinned oracle (oracle/specflow_oracle.py),
fp64 at 1e-12 and the fp32 mode at 1e-5: the fused verify (draft values given,
K <= 8), the generic K > 8 route (device interpolation + per-branch field
evaluations + device epilogue, verifier.py:132-135), the fused speculative
round with the draft MLP, and the Euler full path (flowpolicy.py:273-292)."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

RTOL = {"fp64": 1e-12, "fp32": 1e-5}


def _models(h, d, seed):
    from paper_2605_13778_b200.actions import ChannelLayout
    from paper_2605_13778_b200.flowpolicy import VelocityField
    from paper_2605_13778_b200.nets import init_mlp

    lay = ChannelLayout(3, d - 4)
    rng = np.random.default_rng(seed)
    field_net = init_mlp([h * d + 1 + 39 + 3, 128, 128, h * d], rng)
    draft_net = init_mlp([10, 96, 96, h * d], rng)
    field = VelocityField(net=field_net, horizon=h, dim=d, emb_dim=39, state_dim=3, layout=lay)
    return field, field_net, draft_net, lay, rng


def _ws(net):
    return [np.asarray(w) for w in net.weights], [np.asarray(b) for b in net.biases]


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("h", [16, 50, 100])
@pytest.mark.parametrize("k", [1, 2, 4, 8, 12])
def test_verify_sweep_matches_oracle(prec, h, k):
    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import precision
    from paper_2605_13778_b200.actions import STANDARDIZED, ActionChunk
    from paper_2605_13778_b200.flowpolicy import ConditioningCache
    from paper_2605_13778_b200.verifier import VerifierConfig, verify

    d = 7
    field, field_net, _, lay, rng = _models(h, d, 100 * h + k)
    fw, fb = _ws(field_net)
    taus = tuple((i + 1) / (k + 1) for i in range(k))
    vals = rng.standard_normal((h, d))
    vals[:, -1] = np.abs(vals[:, -1]) + 0.1  # one-signed gripper: the gate depends on the sign
    emb, state = rng.standard_normal(39), rng.standard_normal(3)
    for metric, sign, window in (("l2", -1.0, None), ("linf", 1.0, 12)):
        # delta at the median deciding distance so prefixes vary
        eps = np.random.default_rng(7).standard_normal((h, d))
        probe = so.verify(lambda x, t: so.mlp_field_velocity(fw, fb, x, t, emb, state), vals, eps, taus, 1e9,
                          lay.continuous_dims, metric, window, sign)
        delta = float(np.median(probe["distances"]))
        cfg = VerifierConfig(timesteps=taus, delta=delta, metric=metric, gripper_window=window)
        with precision(prec):
            rep = verify(field, ActionChunk(vals, lay, STANDARDIZED), ConditioningCache(emb), state, cfg,
                         np.random.default_rng(7), current_gripper_sign=sign)
        ref = so.verify(lambda x, t: so.mlp_field_velocity(fw, fb, x, t, emb, state), vals, eps, taus, delta,
                        lay.continuous_dims, metric, window, sign)
        r = RTOL[prec]
        np.testing.assert_allclose(rep.reconstructed, ref["reconstructed"], rtol=r, atol=r)
        np.testing.assert_allclose(rep.distances, ref["distances"], rtol=r, atol=r)
        assert rep.gripper_switch_detected == ref["gripper_switch_detected"]
        margin = np.abs(ref["distances"] - delta).min()
        if rep.branch_prefixes != tuple(ref["branch_prefixes"]):
            assert margin < 1e-4, "decision flip outside the 1e-4 exemption band"
        else:
            assert rep.prefix == ref["prefix"]


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("h,k", [(16, 1), (50, 4), (100, 8)])
def test_flash_round_and_full_round_sweep(prec, h, k):
    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import precision
    from paper_2605_13778_b200.flowpolicy import ConditioningCache, DenoiseConfig, integrate_flow
    from paper_2605_13778_b200.verifier import VerifierConfig, tiny_flash_round

    d = 7
    field, field_net, draft_net, lay, rng = _models(h, d, 7 * h + k)
    fw, fb = _ws(field_net)
    dw, db = _ws(draft_net)
    taus = tuple((i + 1) / (k + 1) for i in range(k))
    feats, emb, state = rng.standard_normal(10), rng.standard_normal(39), rng.standard_normal(3)
    eps = rng.standard_normal((h, d))
    cfg = VerifierConfig(timesteps=taus, delta=1.0, gripper_window=24)
    r = RTOL[prec]
    with precision(prec):
        vals, rep = tiny_flash_round(field, draft_net, feats, ConditioningCache(emb), state, eps, cfg, -1.0, lay)
        full = integrate_flow(field, ConditioningCache(emb), state, DenoiseConfig(10), np.random.default_rng(3))
    dv = so.propose(dw, db, feats, h, d)
    ref = so.verify(lambda x, t: so.mlp_field_velocity(fw, fb, x, t, emb, state), dv, eps, taus, 1.0,
                    lay.continuous_dims, "l2", 24, -1.0)
    np.testing.assert_allclose(vals, dv, rtol=r, atol=r)
    np.testing.assert_allclose(rep.reconstructed, ref["reconstructed"], rtol=r, atol=r)
    np.testing.assert_allclose(rep.distances, ref["distances"], rtol=r, atol=r)
    want = so.integrate_flow(lambda x, t: so.mlp_field_velocity(fw, fb, x, t, emb, state),
                             np.random.default_rng(3).standard_normal((h, d)), 10)
    np.testing.assert_allclose(full, want, rtol=10 * r, atol=10 * r)
