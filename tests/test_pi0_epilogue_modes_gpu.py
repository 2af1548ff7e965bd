"""pi0-scale verify epilogue modes vs the reference's decision rule, in the
fp32 mode of the layer stack (``precision="fp32"``, north-star rtol 1e-5):
metric l2 / linf (actions.py:168-181), gripper window None / 0 / 6
(actions.py:193-211) and delta at 0, at the median deciding distance and
beyond every distance (verifier.py:94-106). The oracle is the unrounded fp32
numpy model (oracle/pi0_oracle.py, bf16_points=False) driving the pinned
reference restatement (oracle/specflow_oracle.py). Decisions must be
identical except when a distance lies within 1e-4 of delta (none expected)."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

SMALL = dict(width=512, layers=2, q_heads=8, head_dim=256, mlp=1024, action_dim=8, state_dim=8,
             horizon=10, prefix_len=200)


@pytest.fixture(scope="module")
def setup():
    from oracle import pi0_oracle as po
    from paper_2605_13778_b200 import pi0

    ocfg, dcfg = po.AEConfig(**SMALL), pi0.AEConfig(**SMALL)
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=2, kv_seed=1, precision="fp32")
    w = po.make_weights(ocfg, 0)
    kvs = [po.make_prefix_kv(ocfg, 1, e) for e in range(2)]
    rng = np.random.default_rng(42)
    H, D, S = SMALL["horizon"], SMALL["action_dim"], SMALL["state_dim"]
    draft = rng.standard_normal((2, H, D)).astype(np.float32)
    draft[:, :, -1] = np.abs(draft[:, :, -1]) + 0.5  # one-signed gripper column
    draft[1, 3, -1] = -0.7                           # env 1: a switch at row 3
    eps = rng.standard_normal((2, H, D)).astype(np.float32)
    state = rng.standard_normal((2, S)).astype(np.float32)
    return ocfg, ae, w, kvs, draft, eps, state


@pytest.mark.parametrize("metric", ["l2", "linf"])
@pytest.mark.parametrize("window", [None, 0, 6])
def test_epilogue_modes_match_reference_rule(setup, metric, window):
    import torch

    from oracle import pi0_oracle as po
    from oracle import specflow_oracle as so
    from paper_2605_13778_b200.verifier import VerifierConfig

    ocfg, ae, w, kvs, draft, eps, state = setup
    taus = (0.25, 0.5, 0.75)
    D = SMALL["action_dim"]
    signs = np.array([1.0, 1.0], np.float32)
    refs = []
    for e in range(2):
        def vel(x, tau, e=e):
            return po.field_velocity(ocfg, w, kvs[e], [(x.astype(np.float32), tau)], state[e],
                                     bf16_points=False)[0]
        refs.append(lambda delta, e=e, vel=vel: so.verify(
            vel, draft[e].astype(np.float64), eps[e].astype(np.float64), taus, delta, D - 1, metric, window,
            float(signs[e])))
    probe = [r(1e9) for r in refs]
    med = float(np.median(np.concatenate([p["distances"].ravel() for p in probe])))
    cuda = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    for delta in (0.0, med, 1e9):
        cfg = VerifierConfig(timesteps=taus, delta=delta, metric=metric, gripper_window=window)
        recon, dist, branch, result = ae.verify_batch(cfg, cuda(draft), cuda(eps), cuda(state), cuda(signs))
        recon, dist = recon.double().cpu().numpy(), dist.double().cpu().numpy()
        branch, result = branch.cpu().numpy(), result.cpu().numpy()
        for e in range(2):
            ref = probe[e] if delta == 1e9 else refs[e](delta)
            np.testing.assert_allclose(recon[e], ref["reconstructed"], rtol=1e-4, atol=1e-4)
            np.testing.assert_allclose(dist[e], ref["distances"], rtol=1e-4, atol=1e-4)
            assert np.abs(ref["distances"] - delta).min() >= 1e-4 or delta == 0.0
            assert tuple(int(x) for x in branch[e]) == tuple(ref["branch_prefixes"])
            assert int(result[e, 0]) == ref["prefix"]
            assert bool(result[e, 1]) == ref["gripper_switch_detected"]
            path, planned = so.fallback_decision(ref["prefix"], ref["gripper_switch_detected"],
                                                 SMALL["horizon"])
            assert ("flash_accepted", "flash_rejected_fallback", "flash_phase_fallback")[result[e, 2]] == path
            assert int(result[e, 3]) == planned
        if delta == 0.0:
            assert (result[:, 0] == 0).all()  # every distance > 0: nothing accepted
        if delta == 1e9:
            assert (result[:, 0] == SMALL["horizon"]).all()
