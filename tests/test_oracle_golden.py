"""Pin the CPU oracle against golden vectors produced by the REAL reference.

The oracle (oracle/specflow_oracle.py) is the checker for every GPU parity
test; here it must reproduce the reference's own outputs (cfg1 random-init
rounds, and every verify / full round of 13 trained-model cfg2 episodes).
"""

import numpy as np
import pytest

from oracle import specflow_oracle as so
from tiny_models import cfg1_golden, cfg1_numpy_weights, cfg2_models, cfg2_trace


def _checksum(a):
    a = np.asarray(a, np.float64)
    return np.array([a.sum(), (a * a).sum(), a.ravel()[0], a.ravel()[-1]])


@pytest.fixture(scope="module")
def g1():
    return cfg1_golden()


def test_cfg1_weights_regenerate_exactly(g1):
    enc, field, draft = cfg1_numpy_weights(g1)
    for name, (ws, _) in (("enc", enc), ("field", field), ("draft", draft)):
        got = np.stack([_checksum(w) for w in ws])
        assert np.array_equal(got, g1[f"{name}_checksums"]), name


def test_cfg1_oracle_matches_reference(g1):
    (ew, eb), (fw, fb), (dw, db) = cfg1_numpy_weights(g1)
    h = int(g1["h"])
    pos, rot = (int(x) for x in g1["layout"])
    d, c = pos + rot + 1, pos + rot
    taus = tuple(g1["taus"])
    n = len(g1["case_vseed"])
    for i in range(n):
        feats = so.draft_features(g1["case_world"][i], int(g1["case_task"][i]), 2,
                                  g1["case_robot_state"][i])
        draft = so.propose(dw, db, feats, h, d)
        if i % 3 != 1:  # make_golden forced a one-signed gripper on these cases
            np.testing.assert_allclose(draft, g1["case_draft"][i], rtol=0, atol=1e-13)
        emb = so.encode_context(ew, eb, feats[:7])
        np.testing.assert_allclose(emb, g1["case_emb"][i], rtol=0, atol=1e-13)
        eps = np.random.default_rng(int(g1["case_vseed"][i])).standard_normal((h, d))
        assert np.array_equal(eps, g1["case_eps"][i])
        state = g1["case_state"][i]

        def vel(x, tau):
            return so.mlp_field_velocity(fw, fb, x, tau, emb, state)

        metric = "l2" if int(g1["case_metric"][i]) == 0 else "linf"
        win = int(g1["case_window"][i])
        rep = so.verify(vel, g1["case_draft"][i], eps, taus, float(g1["case_delta"][i]), c, metric,
                        None if win < 0 else win, float(g1["case_sign"][i]))
        np.testing.assert_allclose(rep["reconstructed"], g1["case_recon"][i], rtol=0, atol=1e-12)
        np.testing.assert_allclose(rep["distances"], g1["case_distances"][i], rtol=0, atol=1e-12)
        assert rep["branch_prefixes"] == tuple(g1["case_branch"][i])
        assert rep["prefix"] == int(g1["case_prefix"][i])
        assert rep["gripper_switch_detected"] == bool(g1["case_switch"][i])
        start = np.random.default_rng(int(g1["case_dseed"][i])).standard_normal((h, d))
        full = so.integrate_flow(vel, start, 10)
        np.testing.assert_allclose(full, g1["case_full"][i], rtol=0, atol=1e-12)


def test_cfg1_golden_exercises_all_branches(g1):
    # acceptance coverage: some rounds accept, some reject (random-init
    # reconstructions flip the gripper in every round, so the gate's negative
    # branch is covered by the trained cfg2 trace instead)
    assert (g1["case_prefix"] == 0).any() and (g1["case_prefix"] > 0).any()
    assert g1["case_switch"].any()


def test_cfg2_trace_gate_fires_both_ways(trace):
    sw = trace["call_switch"][trace["call_kind"] == 1].astype(bool)
    assert sw.any() and (~sw).any()


@pytest.fixture(scope="module")
def trace():
    return cfg2_trace()


def test_cfg2_oracle_replays_reference_trace(trace):
    enc, field, std, draft = cfg2_models()
    fw = [np.asarray(w) for w in field.net.weights]
    fb = [np.asarray(b) for b in field.net.biases]
    dw = [np.asarray(w) for w in draft.net.weights]
    db = [np.asarray(b) for b in draft.net.biases]
    ew = [np.asarray(w) for w in enc.net.weights]
    eb = [np.asarray(b) for b in enc.net.biases]
    h, d = field.horizon, field.dim
    c = field.layout.continuous_dims
    taus = tuple(trace["taus"])
    delta, window = float(trace["delta"]), int(trace["window"])
    n_steps = int(trace["num_steps"])
    kinds = trace["call_kind"]
    n_verify = 0
    for i in range(len(kinds)):
        emb, state = trace["call_emb"][i], trace["call_state"][i]

        def vel(x, tau):
            return so.mlp_field_velocity(fw, fb, x, tau, emb, state)

        seed = int(trace["call_seed"][i])
        if kinds[i] == 1:
            n_verify += 1
            dv = so.propose(dw, db, trace["call_dfeat"][i], h, d)
            np.testing.assert_allclose(dv, trace["call_draft"][i], rtol=0, atol=1e-12)
            eps = np.random.default_rng(seed).standard_normal((h, d))
            rep = so.verify(vel, trace["call_draft"][i], eps, taus, delta, c, "l2", window,
                            float(trace["call_sign"][i]))
            np.testing.assert_allclose(rep["distances"], trace["call_distances"][i], rtol=0,
                                       atol=1e-12)
            assert rep["branch_prefixes"] == tuple(trace["call_branch"][i])
            assert rep["gripper_switch_detected"] == bool(trace["call_switch"][i])
        else:
            emb2 = so.encode_context(ew, eb, trace["call_efeat"][i])
            np.testing.assert_allclose(emb2, emb, rtol=0, atol=1e-13)
            start = np.random.default_rng(seed).standard_normal((h, d))
            out = so.integrate_flow(vel, start, n_steps)
            np.testing.assert_allclose(out, trace["call_chunk"][i], rtol=0, atol=1e-12)
    assert n_verify > 300


def test_cfg2_trace_covers_every_path(trace):
    names = list(trace["path_names"])
    for p in ("flash_accepted", "flash_phase_fallback", "flash_rejected_fallback", "full",
              "periodic_refresh"):
        assert p in names


def test_cfg2_decisions_follow_oracle_rule(trace):
    """Every flash round's recorded path/planned equals the oracle decision rule
    applied to the recorded verifier outputs (runtime.py:286-320)."""
    names = list(trace["path_names"])
    flash = trace["call_kind"] == 1
    ep_c, rd_c = trace["call_episode"][flash], trace["call_round"][flash]
    pre_c, sw_c = trace["call_branch"][flash].min(axis=1), trace["call_switch"][flash]
    lookup = {(int(e), int(r)): (int(p), bool(s)) for e, r, p, s in zip(ep_c, rd_c, pre_c, sw_c)}
    checked = 0
    for e, r, path, planned in zip(trace["round_episode"], trace["round_round"], trace["round_path"],
                                   trace["round_planned"]):
        key = (int(e), int(r))
        if key not in lookup:
            continue
        pre, sw = lookup[key]
        want_path, want_planned = so.fallback_decision(pre, sw, 50, True, True,
                                                       int(trace["replan_size"]))
        assert names[int(path)] == want_path
        assert int(planned) == want_planned
        checked += 1
    assert checked == int(flash.sum())
