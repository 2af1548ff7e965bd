"""Ports of the reference's verifier / Euler known-answer tests
(tests/test_verifier.py:118-258, tests/test_flowpolicy.py:80-163,
bench/selftest.py:36-116) run against the device path. Closed-form fields are
evaluated on the host; interpolation, reconstruction, distances, prefix scan,
gate and Euler updates run in the library's kernels."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _mods():
    from paper_2605_13778_b200 import actions, flowpolicy, verifier

    return actions, flowpolicy, verifier


def _setup():
    actions, flowpolicy, verifier = _mods()
    layout = actions.ChannelLayout(2, 0)
    cache = flowpolicy.ConditioningCache(np.zeros(0))
    return layout, cache, np.zeros(0)


def std_chunk(values, layout):
    from paper_2605_13778_b200.actions import STANDARDIZED, ActionChunk

    return ActionChunk(np.asarray(values, float), layout, STANDARDIZED)


def offset_field(draft_values, offsets, layout):
    from paper_2605_13778_b200.flowpolicy import AnalyticField

    goal = np.asarray(draft_values, float) + np.asarray(offsets, float)
    return AnalyticField(fn=lambda v, t: (goal - v) / (1.0 - t), horizon=goal.shape[0],
                         dim=goal.shape[1], layout=layout)


def test_interpolate_endpoints():
    _, _, verifier = _mods()
    rng = np.random.default_rng(0)
    a, e = rng.normal(size=(2, 4, 3))
    assert np.array_equal(verifier.interpolate(a, e, 0.0), e)
    assert np.array_equal(verifier.interpolate(a, e, 1.0), a)
    with pytest.raises(ValueError):
        verifier.interpolate(np.zeros((2, 3)), np.zeros((3, 3)), 0.5)


def test_reconstruct_oracle_field_recovers_draft():
    _, flowpolicy, verifier = _mods()
    layout, cache, state = _setup()
    rng = np.random.default_rng(1)
    draft, eps = rng.normal(size=(2, 6, 3))
    field = flowpolicy.straight_line_field(draft, layout=layout)
    for tau in (0.2, 1 / 3, 2 / 3, 0.9):
        recon = verifier.reconstruct_endpoint(field, draft, eps, tau, cache, state)
        assert np.max(np.abs(recon - draft)) <= 1e-12
    with pytest.raises(ValueError):
        verifier.reconstruct_endpoint(field, draft, eps, 1.0, cache, state)


def test_oracle_field_accepts_everything():
    _, flowpolicy, verifier = _mods()
    layout, cache, state = _setup()
    draft = std_chunk(np.random.default_rng(3).normal(size=(10, 3)), layout)
    field = flowpolicy.straight_line_field(draft.values, layout=layout)
    rep = verifier.verify(field, draft, cache, state, verifier.VerifierConfig(),
                          np.random.default_rng(0))
    assert rep.prefix == 10 and float(rep.distances.max()) <= 1e-9


def test_selftest_oracle_verify_100_cases():
    """bench/selftest.py:53-74: K in {1,2,4}, H=50, delta=1e-12 -> prefix = H."""
    _, flowpolicy, verifier = _mods()
    layout, cache, state = _setup()
    rng = np.random.default_rng(7)
    worst = 0.0
    for case in range(100):
        k = int(rng.choice([1, 2, 4]))
        taus = tuple(np.sort(rng.uniform(0.05, 0.95, size=k)))
        vals = rng.standard_normal((50, 3))
        field = flowpolicy.straight_line_field(vals, layout=layout)
        rep = verifier.verify(field, std_chunk(vals, layout), cache, state,
                              verifier.VerifierConfig(timesteps=taus, delta=1e-12),
                              np.random.default_rng(np.random.SeedSequence([7, case])))
        worst = max(worst, float(rep.distances.max()))
        assert rep.prefix == 50
    assert worst <= 1e-9


def test_conservative_minimum_over_branches():
    _, flowpolicy, verifier = _mods()
    layout, cache, state = _setup()
    rng = np.random.default_rng(4)
    draft = std_chunk(rng.normal(size=(10, 3)), layout)

    def fn(values, tau):
        goal = draft.values.copy()
        goal[(7 if tau < 0.5 else 3):, :2] += 1.0
        return (goal - values) / (1.0 - tau)

    field = flowpolicy.AnalyticField(fn=fn, horizon=10, dim=3, layout=layout)
    rep = verifier.verify(field, draft, cache, state, verifier.VerifierConfig(delta=0.15),
                          np.random.default_rng(1))
    assert rep.branch_prefixes == (7, 3) and rep.prefix == 3


def test_zero_delta_rejects():
    _, _, verifier = _mods()
    layout, cache, state = _setup()
    draft = std_chunk(np.random.default_rng(5).normal(size=(5, 3)), layout)
    off = np.zeros((5, 3))
    off[:, 0] = 0.01
    rep = verifier.verify(offset_field(draft.values, off, layout), draft, cache, state,
                          verifier.VerifierConfig(delta=0.0), np.random.default_rng(2))
    assert rep.prefix == 0
    # random gripper column flips sign -> the phase label wins (runtime.py:291)
    assert rep.decision == ("flash_phase_fallback" if rep.gripper_switch_detected
                            else "flash_rejected_fallback")


def test_gripper_only_disagreement_and_branch_switch():
    _, _, verifier = _mods()
    layout, cache, state = _setup()
    vals = np.random.default_rng(6).normal(size=(5, 3))
    vals[:, 2] = -1.0
    draft = std_chunk(vals, layout)
    off = np.zeros((5, 3))
    off[:, 2] = -0.5
    rep = verifier.verify(offset_field(vals, off, layout), draft, cache, state,
                          verifier.VerifierConfig(delta=1e-9), np.random.default_rng(3), -1.0)
    assert rep.prefix == 5 and not rep.gripper_switch_detected
    vals = np.random.default_rng(7).normal(size=(6, 3))
    vals[:, 2] = -0.8
    off = np.zeros((6, 3))
    off[4, 2] = 1.6
    rep = verifier.verify(offset_field(vals, off, layout), std_chunk(vals, layout), cache, state,
                          verifier.VerifierConfig(delta=0.15), np.random.default_rng(4), -1.0)
    assert rep.gripper_switch_detected and rep.prefix == 6
    assert rep.decision == "flash_phase_fallback"


def test_shared_noise_determinism_and_eval_count():
    _, flowpolicy, verifier = _mods()
    layout, cache, state = _setup()
    rng = np.random.default_rng(8)
    draft = std_chunk(rng.normal(size=(8, 3)), layout)
    field = offset_field(draft.values, rng.normal(size=(8, 3)) * 0.1, layout)
    cfg = verifier.VerifierConfig(delta=0.1)
    a = verifier.verify(field, draft, cache, state, cfg, np.random.default_rng(42), noise_seed=42)
    b = verifier.verify(field, draft, cache, state, cfg, np.random.default_rng(42), noise_seed=42)
    assert np.array_equal(a.distances, b.distances) and a.branch_prefixes == b.branch_prefixes
    assert a.shared_noise_seed == 42
    sl = flowpolicy.straight_line_field(draft.values, layout=layout)
    for k, taus in ((1, (0.5,)), (2, (1 / 3, 2 / 3)), (4, (0.2, 0.4, 0.6, 0.8))):
        sl.eval_count = 0
        verifier.verify(sl, draft, cache, state, verifier.VerifierConfig(timesteps=taus),
                        np.random.default_rng(0))
        assert sl.eval_count == k


def test_raw_draft_rejected():
    from paper_2605_13778_b200.actions import ActionChunk

    _, flowpolicy, verifier = _mods()
    layout, cache, state = _setup()
    chunk = ActionChunk(np.zeros((2, 3)), layout, "raw")
    with pytest.raises(ValueError):
        verifier.verify(flowpolicy.straight_line_field(np.zeros((2, 3)), layout), chunk, cache,
                        state, verifier.VerifierConfig(), np.random.default_rng(0))


@given(st.integers(0, 2 ** 32 - 1))
@settings(max_examples=15, deadline=None)
def test_monotone_in_delta_and_timesteps(seed):
    _, _, verifier = _mods()
    layout, cache, state = _setup()
    rng = np.random.default_rng(seed)
    draft = std_chunk(rng.normal(size=(6, 3)), layout)
    field = offset_field(draft.values, rng.normal(size=(6, 3)) * 0.15, layout)
    d1, d2 = sorted(rng.uniform(0.0, 0.4, size=2))
    l1 = verifier.verify(field, draft, cache, state, verifier.VerifierConfig(delta=float(d1)),
                         np.random.default_rng(seed)).prefix
    l2 = verifier.verify(field, draft, cache, state, verifier.VerifierConfig(delta=float(d2)),
                         np.random.default_rng(seed)).prefix
    assert l1 <= l2
    small = verifier.VerifierConfig(timesteps=(1 / 3, 2 / 3), delta=0.15)
    large = verifier.VerifierConfig(timesteps=(0.2, 1 / 3, 2 / 3, 0.9), delta=0.15)
    ls = verifier.verify(field, draft, cache, state, small, np.random.default_rng(seed)).prefix
    ll = verifier.verify(field, draft, cache, state, large, np.random.default_rng(seed)).prefix
    assert ll <= ls


@pytest.mark.parametrize("n", [1, 2, 7, 10])
def test_constant_field_euler_exact(n):
    _, flowpolicy, _ = _mods()
    layout, cache, state = _setup()
    c = np.random.default_rng(5).standard_normal((3, 3))
    start = np.random.default_rng(123).standard_normal((3, 3))
    out = flowpolicy.integrate_flow(flowpolicy.constant_field(c, layout), cache, state,
                                    flowpolicy.DenoiseConfig(n), np.random.default_rng(123))
    assert np.max(np.abs(out - (start + c))) <= 1e-12


@pytest.mark.parametrize("n", [1, 3, 10])
def test_straight_line_hits_target(n):
    _, flowpolicy, _ = _mods()
    layout, cache, state = _setup()
    target = np.random.default_rng(6).standard_normal((5, 3))
    out = flowpolicy.integrate_flow(flowpolicy.straight_line_field(target, layout), cache, state,
                                    flowpolicy.DenoiseConfig(n), np.random.default_rng(7))
    assert np.max(np.abs(out - target)) <= 1e-9


def test_divergence_reports_tau():
    _, flowpolicy, _ = _mods()
    layout, cache, state = _setup()
    field = flowpolicy.AnalyticField(fn=lambda v, t: np.full_like(v, np.nan), horizon=2, dim=3,
                                     layout=layout)
    with pytest.raises(FloatingPointError, match="tau"):
        flowpolicy.integrate_flow(field, cache, state, flowpolicy.DenoiseConfig(4),
                                  np.random.default_rng(0))


def test_zero_net_velocity_and_propose():
    """test_flowpolicy.py:80-92 and test_draft.py:45-67 on the device MLP kernels."""
    from paper_2605_13778_b200.draft import DraftModel, propose
    from paper_2605_13778_b200.flowpolicy import (ObsNormalizer, Observation, VelocityField,
                                                  velocity)
    from paper_2605_13778_b200.nets import Mlp, init_mlp

    layout, cache, state = _setup()
    h, d = 4, 3
    net = Mlp(weights=[np.zeros((h * d, h * d + 1))], biases=[np.zeros(h * d)])
    field = VelocityField(net=net, horizon=h, dim=d, emb_dim=0, state_dim=0, layout=layout)
    assert np.array_equal(velocity(field, np.zeros((h, d)), 0.5, cache, state), np.zeros((h, d)))
    assert np.allclose(velocity(field, np.ones((h, d)), 0.5, cache, state), -2.0)
    model = DraftModel(net=init_mlp([7, 16, 4 * 3], np.random.default_rng(0)), layout=layout,
                       horizon=4, n_tasks=2, normalizer=ObsNormalizer.identity(3, 2))
    for w in model.net.weights:
        w[...] = 0.0
    model.net.invalidate_device()
    obs = Observation(np.zeros(3), 0, np.zeros(2))
    assert np.array_equal(propose(model, obs).values, np.zeros((4, 3)))
    m2 = DraftModel(net=init_mlp([7, 16, 50 * 3], np.random.default_rng(3)), layout=layout,
                    horizon=50, n_tasks=2, normalizer=ObsNormalizer.identity(3, 2))
    o2 = Observation(np.array([1.0, -1.0, 2.0]), 1, np.array([0.5, 0.1]))
    a, b = propose(m2, o2), propose(m2, o2)
    assert a.horizon == 50 and np.array_equal(a.values, b.values)
    with pytest.raises(ValueError):
        propose(m2, Observation(np.zeros(3), 5, np.zeros(2)))
