"""The reference-facing plugin calls on the pi0-scale field: the reference's
``verifier.verify(field, draft, cache, state, cfg, rng)`` (verifier.py:109-150)
and ``flowpolicy.integrate_flow(field, cache, state, cfg, rng)``
(flowpolicy.py:273-292) with the ActionExpert as the field, numpy in / numpy
out. They must equal the device-tensor entry points on the same inputs and
draw the noise from the caller's rng exactly once (verifier.py:129,
flowpolicy.py:286)."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

SMALL = dict(width=512, layers=2, q_heads=8, head_dim=256, mlp=1024, action_dim=8, state_dim=8,
             horizon=10, prefix_len=200)


def _setup():
    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.actions import STANDARDIZED, ActionChunk
    from paper_2605_13778_b200.flowpolicy import ConditioningCache

    ae = pi0.ActionExpert(pi0.AEConfig(**SMALL), seed=0, n_envs=1, kv_seed=1)
    rng = np.random.default_rng(11)
    vals = rng.standard_normal((SMALL["horizon"], SMALL["action_dim"]))
    draft = ActionChunk(values=vals, layout=ae.layout, space=STANDARDIZED)
    state = rng.standard_normal(SMALL["state_dim"])
    return ae, draft, ConditioningCache(embedding=np.zeros(0), kv=0), state


@pytest.mark.parametrize("sign", [-1.0, 1.0])
def test_plugin_verify_equals_device_verify(sign):
    import torch

    from paper_2605_13778_b200.verifier import VerifierConfig, verify

    ae, draft, cache, state = _setup()
    cfg = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=2.0, gripper_window=None)
    rep = verify(ae, draft, cache, state, cfg, np.random.default_rng(5), current_gripper_sign=sign, noise_seed=5)
    eps = np.random.default_rng(5).standard_normal(draft.values.shape)
    f32 = lambda a: torch.from_numpy(np.asarray(a, np.float32)).cuda()  # noqa: E731
    recon, dist, branch, result = ae.verify_batch(cfg, f32(draft.values)[None], f32(eps)[None],
                                                  f32(state)[None], current_sign=sign)
    torch.cuda.synchronize()
    res = result[0].cpu().numpy()
    assert np.array_equal(rep.reconstructed, recon[0].double().cpu().numpy())
    assert np.array_equal(rep.distances, dist[0].double().cpu().numpy())
    assert rep.branch_prefixes == tuple(int(x) for x in branch[0].cpu())
    assert rep.prefix == int(res[0]) and rep.gripper_switch_detected == bool(res[1])
    assert rep.shared_noise_seed == 5 and rep.reconstructed.shape == (4,) + draft.values.shape
    assert ae.eval_count == 4


def test_plugin_integrate_flow_equals_device_denoise():
    import torch

    from paper_2605_13778_b200.flowpolicy import DenoiseConfig, integrate_flow

    ae, _, cache, state = _setup()
    got = integrate_flow(ae, cache, state, DenoiseConfig(num_steps=6), np.random.default_rng(9))
    a0 = np.random.default_rng(9).standard_normal((SMALL["horizon"], SMALL["action_dim"]))
    f32 = lambda a: torch.from_numpy(np.asarray(a, np.float32)).cuda()  # noqa: E731
    chunk, status = ae.denoise_batch(f32(a0)[None], f32(state)[None], 6)
    torch.cuda.synchronize()
    assert status[0, 0].item() == -1
    assert np.array_equal(got, chunk[0].double().cpu().numpy())
    assert ae.eval_count == 6
