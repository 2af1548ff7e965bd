"""pi0-scale Action Expert on the device vs the numpy oracle (oracle/pi0_oracle.py).

Reduced shapes check the whole chain element-wise (both GEMM orientations,
split-K / split-KV attention, batched envs); the full cfg3 shape is checked
against the oracle at the north-star bf16 tolerance (rtol 1e-2) and by
size-independent properties (determinism, graph == eager, batched == single).
"""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

SMALL = dict(width=512, layers=2, q_heads=8, head_dim=256, mlp=1024, action_dim=8, state_dim=8,
             horizon=10, prefix_len=200)


def _pair(**over):
    from oracle import pi0_oracle as po
    from paper_2605_13778_b200 import pi0

    kw = dict(SMALL, **over)
    return po.AEConfig(**kw), pi0.AEConfig(**kw)


def test_hash_init_matches_oracle_bitwise():
    import torch

    from oracle import pi0_oracle as po
    from paper_2605_13778_b200 import pi0

    for dtype, conv in ((torch.float32, lambda a: a), (torch.bfloat16, po.bf16)):
        t = pi0._fill(torch.empty((37, 129), dtype=dtype, device="cuda"), 5, 123, 0.02)
        want = conv(po.hash_uniform(5, 123, (37, 129), 0.02))
        assert np.array_equal(t.float().cpu().numpy(), want)


def _oracle_weights(ocfg, seed=0, kv_seed=1, env=0):
    from oracle import pi0_oracle as po

    return po.make_weights(ocfg, seed), po.make_prefix_kv(ocfg, kv_seed, env)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_velocity_matches_oracle_small(k):
    import torch

    from oracle import pi0_oracle as po
    from paper_2605_13778_b200 import pi0

    ocfg, dcfg = _pair()
    w, kv = _oracle_weights(ocfg)
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=1, kv_seed=1)
    rng = np.random.default_rng(k)
    taus = [(i + 1) / (k + 1) for i in range(k)]
    xs = rng.standard_normal((k, dcfg.horizon, dcfg.action_dim)).astype(np.float32)
    state = rng.standard_normal(dcfg.state_dim).astype(np.float32)
    got = ae.velocity_batch(torch.from_numpy(xs[None]).cuda(), taus,
                            torch.from_numpy(state[None]).cuda())[0].cpu().numpy()
    want = po.field_velocity(ocfg, w, kv, [(xs[i], taus[i]) for i in range(k)], state)
    np.testing.assert_allclose(got, want, rtol=2e-2, atol=2e-2 * np.abs(want).max())


@pytest.mark.parametrize("n_envs,k", [(1, 4), (3, 2), (6, 4)])
def test_verify_matches_oracle_small(n_envs, k, check_envs=None):
    """Whole verify chain vs the pinned specflow oracle driven by the pi0 oracle
    field; n_envs * env_rows > 256 exercises the batched (normal) GEMM path.
    check_envs: the envs compared against the (slow) oracle (default: all)."""
    import torch

    from oracle import pi0_oracle as po
    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    ocfg, dcfg = _pair()
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=n_envs, kv_seed=1)
    w = po.make_weights(ocfg, 0)
    rng = np.random.default_rng(10 + n_envs)
    H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
    draft = rng.standard_normal((n_envs, H, D)).astype(np.float32)
    eps = rng.standard_normal((n_envs, H, D)).astype(np.float32)
    state = rng.standard_normal((n_envs, S)).astype(np.float32)
    signs = np.where(rng.random(n_envs) < 0.5, -1.0, 1.0).astype(np.float32)
    taus = tuple((i + 1) / (k + 1) for i in range(k))
    cfg = VerifierConfig(timesteps=taus, delta=1.0, gripper_window=6)
    recon, dist, branch, result = ae.verify_batch(
        cfg, torch.from_numpy(draft).cuda(), torch.from_numpy(eps).cuda(),
        torch.from_numpy(state).cuda(), torch.from_numpy(signs).cuda())
    recon, dist = recon.cpu().numpy(), dist.cpu().numpy()
    branch, result = branch.cpu().numpy(), result.cpu().numpy()
    flips = 0
    for e in (range(n_envs) if check_envs is None else check_envs):
        kv = po.make_prefix_kv(ocfg, 1, e)

        def vel(x, tau):
            return po.field_velocity(ocfg, w, kv, [(x.astype(np.float32), tau)], state[e])[0]

        ref = so.verify(vel, draft[e].astype(np.float64), eps[e].astype(np.float64), taus, 1.0,
                        D - 1, "l2", 6, float(signs[e]))
        scale = np.abs(ref["reconstructed"]).max()
        np.testing.assert_allclose(recon[e], ref["reconstructed"], rtol=1e-2, atol=1e-2 * scale)
        np.testing.assert_allclose(dist[e], ref["distances"], rtol=2e-2, atol=2e-2 * scale)
        margin = np.abs(ref["distances"] - 1.0).min()
        if tuple(branch[e]) != ref["branch_prefixes"]:
            assert margin < 5e-2, "prefix flip outside the numerical band"
            flips += 1
        assert bool(result[e, 1]) == ref["gripper_switch_detected"]
        path, planned = so.fallback_decision(int(result[e, 0]), bool(result[e, 1]), H)
        assert ("flash_accepted", "flash_rejected_fallback", "flash_phase_fallback")[result[e, 2]] == path
        assert result[e, 3] == planned
    assert flips <= max(1, n_envs // 3)


def test_verify_matches_oracle_large_batch():
    """200 envs (9600 token rows): the batched kernels' large-M paths (2-SM
    pair attention with one KV split, 8-row embedding CTAs) vs the oracle on a
    few envs."""
    test_verify_matches_oracle_small(200, 4, check_envs=(0, 117, 199))


@pytest.mark.parametrize("attn", ["pair", "single"])
def test_verify_matches_oracle_batched_attention(attn, monkeypatch):
    """The batched (one KV split) attention kernels against the oracle: the
    default 2-SM pair kernel (128-key superblocks, 3 query tiles per env so the
    last pair has a dummy partner) and the 1-SM persistent kernel."""
    monkeypatch.setenv("SF_ATTN_SPLITS", "1")
    if attn == "single":
        monkeypatch.setenv("SF_ATTN_SINGLE", "1")
    else:
        monkeypatch.delenv("SF_ATTN_SINGLE", raising=False)
    test_verify_matches_oracle_small(6, 4)


@pytest.mark.parametrize("n_envs", [1, 300])
def test_flash_round_draft_matches_oracle(n_envs):
    """propose (draft MLP) fused into the verify graph: draft vs oracle, and the
    round's verify outputs equal a verify of that draft."""
    import torch

    from oracle import pi0_oracle as po
    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    ocfg, dcfg = _pair(layers=1, prefix_len=64)
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=n_envs, kv_seed=1)
    rng = np.random.default_rng(n_envs)
    obs = rng.standard_normal((n_envs, dcfg.draft_in)).astype(np.float32)
    eps = rng.standard_normal((n_envs, dcfg.horizon, dcfg.action_dim)).astype(np.float32)
    state = rng.standard_normal((n_envs, dcfg.state_dim)).astype(np.float32)
    cfg = VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=1.0)
    t = lambda a: torch.from_numpy(a).cuda()
    draft, recon, dist, branch, result = [x.clone() for x in ae.flash_batch(cfg, t(obs), t(eps), t(state))]
    want = po.draft_forward(ocfg, po.make_draft_weights(ocfg, 0), obs)
    np.testing.assert_allclose(draft.cpu().numpy(), want, rtol=1e-2, atol=1e-2 * np.abs(want).max())
    r2, d2, b2, res2 = ae.verify_batch(cfg, draft, t(eps), t(state))
    assert torch.equal(r2, recon) and torch.equal(b2, branch) and torch.equal(res2, result)


def test_denoise_matches_oracle_small():
    import torch

    from oracle import pi0_oracle as po
    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import pi0

    ocfg, dcfg = _pair()
    w, kv = _oracle_weights(ocfg)
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=1, kv_seed=1)
    rng = np.random.default_rng(3)
    start = rng.standard_normal((dcfg.horizon, dcfg.action_dim)).astype(np.float32)
    state = rng.standard_normal(dcfg.state_dim).astype(np.float32)
    chunk, status = ae.denoise_batch(torch.from_numpy(start[None]).cuda(),
                                     torch.from_numpy(state[None]).cuda(), 4)
    assert status[0, 0].item() == -1
    want = so.integrate_flow(
        lambda x, t: po.field_velocity(ocfg, w, kv, [(x.astype(np.float32), t)], state)[0], start, 4)
    got = chunk[0].cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=2e-2, atol=2e-2 * np.abs(want).max())


def test_denoise_matches_oracle_large_batch():
    """Euler full path over 300 envs (one 16-row query tile per env: the 1-SM
    persistent attention kernel with one KV split, 8-row embedding CTAs) vs
    the oracle on a few envs."""
    import torch

    from oracle import pi0_oracle as po
    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import pi0

    ocfg, dcfg = _pair()
    E = 300
    w = po.make_weights(ocfg, 0)
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=E, kv_seed=1)
    rng = np.random.default_rng(4)
    start = rng.standard_normal((E, dcfg.horizon, dcfg.action_dim)).astype(np.float32)
    state = rng.standard_normal((E, dcfg.state_dim)).astype(np.float32)
    chunk, status = ae.denoise_batch(torch.from_numpy(start).cuda(), torch.from_numpy(state).cuda(), 4)
    chunk = chunk.cpu().numpy()
    for e in (0, 151, 299):
        kv = po.make_prefix_kv(ocfg, 1, e)
        want = so.integrate_flow(
            lambda x, t: po.field_velocity(ocfg, w, kv, [(x.astype(np.float32), t)], state[e])[0], start[e], 4)
        np.testing.assert_allclose(chunk[e], want, rtol=2e-2, atol=2e-2 * np.abs(want).max())


def test_graph_pdl_matches_eager_and_is_deterministic():
    import torch

    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    _, dcfg = _pair()
    rng = np.random.default_rng(5)
    H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
    d = torch.from_numpy(rng.standard_normal((2, H, D)).astype(np.float32)).cuda()
    e = torch.from_numpy(rng.standard_normal((2, H, D)).astype(np.float32)).cuda()
    s = torch.from_numpy(rng.standard_normal((2, S)).astype(np.float32)).cuda()
    cfg = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=0.5)
    outs = []
    for flags in (0, pi0.SF_AE_GRAPH, pi0.SF_AE_GRAPH | pi0.SF_AE_PDL, pi0.SF_AE_GRAPH | pi0.SF_AE_PDL):
        ae = pi0.ActionExpert(dcfg, seed=0, n_envs=2, kv_seed=1, flags=flags)
        outs.append([t.clone() for t in ae.verify_batch(cfg, d, e, s)])
        outs.append([t.clone() for t in ae.verify_batch(cfg, d, e, s)])
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert torch.equal(a, b)


@pytest.mark.slow
def test_full_size_cfg3_verify_vs_oracle():
    """cfg3: 18 layers, width 1024, P=800, H=50, D=32, K=4, batch 1 — recon
    within the north-star bf16 tolerance (rtol 1e-2); decisions identical
    except rounds within the numerical band of delta."""
    import torch

    from oracle import pi0_oracle as po
    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    ocfg, dcfg = po.AEConfig(), pi0.AEConfig()
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=1, kv_seed=1)
    w, kv = _oracle_weights(ocfg)
    rng = np.random.default_rng(7)
    H, D, S = 50, 32, 32
    draft = rng.standard_normal((1, H, D)).astype(np.float32)
    eps = rng.standard_normal((1, H, D)).astype(np.float32)
    state = rng.standard_normal((1, S)).astype(np.float32)
    taus = (0.2, 0.4, 0.6, 0.8)
    cfg = VerifierConfig(timesteps=taus, delta=4.0, gripper_window=24)
    recon, dist, branch, result = ae.verify_batch(cfg, torch.from_numpy(draft).cuda(),
                                                  torch.from_numpy(eps).cuda(),
                                                  torch.from_numpy(state).cuda())
    ref = so.verify(lambda x, t: po.field_velocity(ocfg, w, kv, [(x.astype(np.float32), t)],
                                                   state[0])[0],
                    draft[0].astype(np.float64), eps[0].astype(np.float64), taus, 4.0, D - 1, "l2",
                    24, -1.0)
    scale = np.abs(ref["reconstructed"]).max()
    np.testing.assert_allclose(recon[0].cpu().numpy(), ref["reconstructed"], rtol=1e-2,
                               atol=1e-2 * scale)
    if tuple(branch[0].cpu().numpy()) != ref["branch_prefixes"]:
        assert np.abs(ref["distances"] - 4.0).min() < 5e-2


def test_attention_pair_kernel_matches_single_sm():
    """Batched rounds (one KV split) run attention on 2-SM CTA pairs by default
    (attn_pair_kernel: 128-key superblocks, odd tile counts paired with a dummy
    partner); it must agree with the 1-SM persistent kernel (SF_ATTN_SINGLE=1)
    on the same inputs."""
    import os

    import torch

    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    _, dcfg = _pair()
    E = 64  # 3 query tiles per env, 192 tiles -> one KV split per tile
    rng = np.random.default_rng(11)
    H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
    d = torch.from_numpy(rng.standard_normal((E, H, D)).astype(np.float32)).cuda()
    e = torch.from_numpy(rng.standard_normal((E, H, D)).astype(np.float32)).cuda()
    s = torch.from_numpy(rng.standard_normal((E, S)).astype(np.float32)).cuda()
    cfg = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=0.5)
    outs = []
    for flag in ("1", None):
        if flag:
            os.environ["SF_ATTN_SINGLE"] = flag
        else:
            os.environ.pop("SF_ATTN_SINGLE", None)
        ae = pi0.ActionExpert(dcfg, seed=0, n_envs=E, kv_seed=1)
        outs.append([t.clone() for t in ae.verify_batch(cfg, d, e, s)])
    os.environ.pop("SF_ATTN_SINGLE", None)
    (r0, d0, _, _), (r1, d1, _, _) = outs
    torch.testing.assert_close(r1, r0, rtol=2e-3, atol=2e-3 * r0.abs().max().item())
    torch.testing.assert_close(d1, d0, rtol=2e-3, atol=2e-3 * d0.abs().max().item())


def _replan_ref(result, fsr, has_cache, mode_flash, pf, r):
    """run_episode bookkeeping (runtime.py:238-320) for one round of B envs."""
    B = len(fsr)
    path, planned, idx = np.zeros(B, int), np.zeros(B, int), []
    fsr, has_cache = fsr.copy(), has_cache.copy()
    for e in range(B):
        forced = pf > 0 and fsr[e] >= pf
        use = mode_flash and has_cache[e] and not forced
        if not use:
            path[e], planned[e] = (4 if (forced and mode_flash) else 3), r
        else:
            path[e] = result[e, 2]
            planned[e] = result[e, 3] if path[e] == 0 else r
        if path[e] == 0:
            fsr[e] += 1
        else:
            fsr[e], has_cache[e] = 0, 1
            idx.append(e)
    return path, planned, fsr, has_cache, np.array(idx, int)


def test_replan_update_matches_run_episode_bookkeeping():
    import torch

    from paper_2605_13778_b200 import _capi

    rng = np.random.default_rng(21)
    B, pf, r = 3000, 2, 12
    for mode_flash in (1, 0):
        result = np.zeros((B, 8), np.int32)
        result[:, 2] = rng.integers(0, 3, B)
        result[:, 3] = rng.integers(1, 13, B)
        fsr = rng.integers(0, 4, B).astype(np.int32)
        hc = rng.integers(0, 2, B).astype(np.int32)
        want = _replan_ref(result, fsr, hc, mode_flash, pf, r)
        t = lambda a: torch.from_numpy(a).cuda()
        d_res, d_fsr, d_hc = t(result), t(fsr), t(hc)
        path, planned, idx = (torch.empty(B, dtype=torch.int32, device="cuda") for _ in range(3))
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        _capi.check(_capi.lib().sf_replan_update(
            B, d_res.data_ptr(), d_fsr.data_ptr(), d_hc.data_ptr(), mode_flash, pf, r, path.data_ptr(),
            planned.data_ptr(), idx.data_ptr(), cnt.data_ptr(), torch.cuda.current_stream().cuda_stream),
            "replan")
        n = int(cnt.item())
        np.testing.assert_array_equal(path.cpu().numpy(), want[0])
        np.testing.assert_array_equal(planned.cpu().numpy(), want[1])
        np.testing.assert_array_equal(d_fsr.cpu().numpy(), want[2])
        np.testing.assert_array_equal(d_hc.cpu().numpy(), want[3])
        np.testing.assert_array_equal(idx[:n].cpu().numpy(), want[4])


def test_denoise_envs_compacted_matches_full_batch():
    import torch

    from paper_2605_13778_b200 import pi0

    _, dcfg = _pair()
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=4, kv_seed=1)
    rng = np.random.default_rng(4)
    H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
    start = torch.from_numpy(rng.standard_normal((4, H, D)).astype(np.float32)).cuda()
    state = torch.from_numpy(rng.standard_normal((4, S)).astype(np.float32)).cuda()
    full, _ = ae.denoise_batch(start, state, 4)
    m = torch.tensor([2, 0], dtype=torch.int32, device="cuda")
    sub, status = ae.denoise_envs(m, start[[2, 0]], state[[2, 0]], 4)
    assert (status[:, 0] == -1).all()
    torch.testing.assert_close(sub, full[[2, 0]], rtol=1e-3, atol=1e-3 * full.abs().max().item())


def test_batched_replanner_rounds():
    import torch

    from paper_2605_13778_b200 import _capi, pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    _, dcfg = _pair()
    B = 6
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=B, kv_seed=1)
    vc = VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=1e9, gripper_window=0)
    rp = pi0.BatchedReplanner(ae, B, vc, replan_size=4, periodic_refresh=2)
    g = torch.Generator(device="cuda").manual_seed(0)
    H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
    mk = lambda *sh: torch.randn(sh, generator=g, device="cuda")
    paths = []
    for _ in range(4):
        obs, ev, ed, st = mk(B, dcfg.draft_in), mk(B, H, D), mk(B, H, D), mk(B, S)
        signs = torch.ones(B, device="cuda")
        chunk, path, planned, _, result = rp.round(obs, ev, ed, st, signs)
        paths.append(path.cpu().numpy().copy())
        p = path.cpu().numpy()
        assert torch.isfinite(chunk).all()
        # accepted envs execute the draft, with the capped prefix
        acc = p == _capi.SF_PATH_FLASH_ACCEPTED
        assert (planned.cpu().numpy()[~acc] == 4).all()
    # round 0: no context yet -> full; delta = inf accepts every flash attempt
    assert (paths[0] == _capi.SF_PATH_FULL).all()
    assert (paths[1] == _capi.SF_PATH_FLASH_ACCEPTED).all()
    assert (paths[2] == _capi.SF_PATH_FLASH_ACCEPTED).all()
    assert (paths[3] == _capi.SF_PATH_PERIODIC).all()  # PF = 2 flash rounds since the refresh


def test_vlm_prefill_matches_oracle_and_feeds_the_expert():
    """Context refresh: prefix encoder K / V written into the
    pool layout, vs the oracle restatement; the pool then drives a verify."""
    import dataclasses

    import torch

    from oracle import pi0_oracle as po
    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    vcfg = pi0.VLMConfig(width=512, layers=2, mlp=1024, prefix_len=96)
    ocfg = po.VLMConfig(width=512, layers=2, mlp=1024, prefix_len=96)
    vlm = pi0.VLMPrefill(vcfg, seed=7)
    E = 2
    rng = np.random.default_rng(8)
    x = rng.standard_normal((E, vcfg.prefix_len, vcfg.width)).astype(np.float32)
    kp, vtp = vlm.prefill(torch.from_numpy(x).cuda())
    layers = po.make_vlm_weights(ocfg, seed=7)
    for e in range(E):
        ks, vts = po.prefill_kv(ocfg, layers, x[e])
        gk = kp[:, e].float().cpu().numpy()
        gv = vtp[:, e].float().cpu().numpy()
        np.testing.assert_allclose(gk, ks, rtol=2e-2, atol=2e-2 * np.abs(ks).max())
        np.testing.assert_allclose(gv, vts, rtol=2e-2, atol=2e-2 * np.abs(vts).max())
    # the refreshed pool is what the Action Expert attends to
    _, dcfg = _pair()
    dcfg = dataclasses.replace(dcfg, prefix_len=vcfg.prefix_len)
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=E, kv_seed=1)
    ae.bind_prefix(kp, vtp)
    H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
    d = torch.from_numpy(rng.standard_normal((E, H, D)).astype(np.float32)).cuda()
    e_ = torch.from_numpy(rng.standard_normal((E, H, D)).astype(np.float32)).cuda()
    s = torch.from_numpy(rng.standard_normal((E, S)).astype(np.float32)).cuda()
    recon, dist, _, _ = ae.verify_batch(VerifierConfig(timesteps=(0.2, 0.6), delta=0.5), d, e_, s)
    assert torch.isfinite(recon).all() and torch.isfinite(dist).all()


def test_prefix_refresh_in_place():
    """A context refresh written INTO the bound pool (VLMPrefill.prefill with
    expert=...) is what the next verify attends to: same outputs as a fresh
    expert bound to the refreshed pool (advisor r1: stale block images)."""
    import dataclasses

    import torch

    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    vcfg = pi0.VLMConfig(width=512, layers=2, mlp=1024, prefix_len=96)
    vlm = pi0.VLMPrefill(vcfg, seed=7)
    E = 2
    rng = np.random.default_rng(9)
    _, dcfg = _pair()
    dcfg = dataclasses.replace(dcfg, prefix_len=vcfg.prefix_len)
    kp, vtp = vlm.prefill(torch.from_numpy(rng.standard_normal((E, 96, 512)).astype(np.float32)).cuda())
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=E, kv_seed=1)
    ae.bind_prefix(kp, vtp)
    H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
    d = torch.from_numpy(rng.standard_normal((E, H, D)).astype(np.float32)).cuda()
    e_ = torch.from_numpy(rng.standard_normal((E, H, D)).astype(np.float32)).cuda()
    s = torch.from_numpy(rng.standard_normal((E, S)).astype(np.float32)).cuda()
    vc = VerifierConfig(timesteps=(0.2, 0.6), delta=0.5)
    before = ae.verify_batch(vc, d, e_, s)[0].clone()
    # refresh in place, then verify again through the same (captured) graph
    vlm.prefill(torch.from_numpy(rng.standard_normal((E, 96, 512)).astype(np.float32)).cuda(), kp, vtp,
                expert=ae)
    after = ae.verify_batch(vc, d, e_, s)[0].clone()
    fresh = pi0.ActionExpert(dcfg, seed=0, n_envs=E, kv_seed=1)
    fresh.bind_prefix(kp.clone(), vtp.clone())
    want = fresh.verify_batch(vc, d, e_, s)[0]
    assert not torch.equal(before, after)
    assert torch.equal(after, want)
