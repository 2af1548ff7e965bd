"""The device replanning round (sf_ae_replan_round / pi0.BatchedReplanner) and
its bookkeeping against the reference's recorded episodes.

* sf_replan_update replays the path / planned sequence of the 13 reference
  cfg2 episodes (run_episode, runtime.py:238-326: periodic refresh PF = 2,
  prefix cap R = 12, phase label over rejection) recorded in
  tests/golden/cfg2_trace.npz;
* one graph-resident round equals its components: flash attempt words, the
  run_episode bookkeeping restated in numpy, the Euler full path of exactly
  the fallback envs (sf_ae_denoise_envs), switch_in_executed
  (runtime.py:321-323) and destandardize (actions.py:139-144).
"""

import numpy as np
import pytest

from conftest import cuda_ok
from tiny_models import cfg2_trace

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

SMALL = dict(width=512, layers=2, q_heads=8, head_dim=256, mlp=1024, action_dim=8, state_dim=8,
             horizon=10, prefix_len=200)
# cfg2_trace path_names order -> device path codes
_TRACE_TO_DEV = {0: 0, 1: 2, 2: 1, 3: 3, 4: 4}


def test_replan_update_replays_reference_episodes():
    """Lock-step replay of the 13 recorded episodes as 13 envs: each round's
    flash words come from the recorded attempt (prefix, switch) through the
    reference decision rule; the device bookkeeping must reproduce the
    recorded path and planned of every round."""
    import torch

    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import _capi

    tr = cfg2_trace()
    ep, rd = tr["round_episode"], tr["round_round"]
    n_env = int(ep.max()) + 1
    n_rounds = int(rd.max()) + 1
    R = int(tr["replan_size"])
    path_t = np.full((n_env, n_rounds), -1)
    plan_t = np.zeros((n_env, n_rounds), int)
    pre_t = np.full((n_env, n_rounds), -1)
    sw_t = np.zeros((n_env, n_rounds), int)
    for i in range(len(ep)):
        e, r = int(ep[i]), int(rd[i])
        path_t[e, r] = _TRACE_TO_DEV[int(tr["round_path"][i])]
        plan_t[e, r] = int(tr["round_planned"][i])
        pre_t[e, r] = int(tr["round_prefix"][i])
        sw_t[e, r] = int(tr["round_switch"][i])
    dev = "cuda"
    fsr = torch.zeros(n_env, dtype=torch.int32, device=dev)
    hc = torch.zeros(n_env, dtype=torch.int32, device=dev)
    out = [torch.empty(n_env, dtype=torch.int32, device=dev) for _ in range(3)]
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    checked = 0
    for r in range(n_rounds):
        words = np.zeros((n_env, 8), np.int32)
        for e in range(n_env):
            if pre_t[e, r] >= 0:  # the reference made a flash attempt this round
                path, planned = so.fallback_decision(int(pre_t[e, r]), bool(sw_t[e, r]), 50, replan_size=R)
                code = ("flash_accepted", "flash_rejected_fallback", "flash_phase_fallback").index(path)
                words[e, :4] = [pre_t[e, r], sw_t[e, r], code, planned]
            else:  # no attempt: words the bookkeeping must ignore (an accepted-looking attempt)
                words[e, :4] = [7, 0, 0, 7]
        d_words = torch.from_numpy(words).to(dev)
        _capi.check(_capi.lib().sf_replan_update(
            n_env, d_words.data_ptr(), fsr.data_ptr(), hc.data_ptr(), 1, 2, R, out[0].data_ptr(),
            out[1].data_ptr(), out[2].data_ptr(), cnt.data_ptr(), torch.cuda.current_stream().cuda_stream),
            "replan")
        got_path, got_plan = out[0].cpu().numpy(), out[1].cpu().numpy()
        for e in range(n_env):
            if path_t[e, r] < 0:
                continue  # the episode ended earlier
            assert got_path[e] == path_t[e, r], (e, r, got_path[e], path_t[e, r])
            assert got_plan[e] == plan_t[e, r], (e, r, got_plan[e], plan_t[e, r])
            checked += 1
    assert checked == len(ep)


def _run_rounds(n, n_rounds, delta, standardizer, seed=0):
    import torch

    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    dcfg = pi0.AEConfig(**SMALL)
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=n, kv_seed=1, draft_gripper_bias=6.0)
    vc = VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=delta, gripper_window=6)
    rp = pi0.BatchedReplanner(ae, n, vc, replan_size=4, periodic_refresh=2, standardizer=standardizer)
    g = torch.Generator(device="cuda").manual_seed(seed)
    H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
    mk = lambda *sh: torch.randn(sh, generator=g, device="cuda")
    rounds = []
    for r in range(n_rounds):
        obs, ev, ed, st = mk(n, dcfg.draft_in), mk(n, H, D), mk(n, H, D), mk(n, S)
        signs = torch.where(torch.arange(n, device="cuda") % 3 == 0, -1.0, 1.0)
        fsr0, hc0 = rp.fsr.clone(), rp.has_cache.clone()
        chunk, path, planned, branch, result = rp.round(obs, ev, ed, st, signs)
        rounds.append(dict(obs=obs, ev=ev, ed=ed, st=st, signs=signs, fsr0=fsr0, hc0=hc0,
                           chunk=chunk.clone(), path=path.clone(), planned=planned.clone(),
                           result=result.clone(), branch=branch.clone(), sie=rp.switch_in_executed.clone(),
                           bad=rp.nonfinite.clone(), nfb=int(rp.n_fallback.item()),
                           raw=rp.chunk_raw.clone() if rp.chunk_raw is not None else None))
    return ae, vc, rp, rounds


def _replan_ref(result, fsr, has_cache, pf, r):
    """run_episode bookkeeping (runtime.py:238-320) for one round of B envs."""
    B = len(fsr)
    path, planned, idx = np.zeros(B, int), np.zeros(B, int), []
    fsr, has_cache = fsr.copy(), has_cache.copy()
    for e in range(B):
        forced = pf > 0 and fsr[e] >= pf
        if not (has_cache[e] and not forced):
            path[e], planned[e] = (4 if forced else 3), r
        else:
            path[e] = result[e, 2]
            planned[e] = result[e, 3] if path[e] == 0 else r
        if path[e] == 0:
            fsr[e] += 1
        else:
            fsr[e], has_cache[e] = 0, 1
            idx.append(e)
    return path, planned, np.array(idx, int)


def test_replan_round_equals_its_components():
    import torch

    from paper_2605_13778_b200.actions import Standardizer

    n = 37
    std = Standardizer(mean=np.linspace(-1, 1, 8), std=np.linspace(0.5, 2.0, 8))
    ae, vc, rp, rounds = _run_rounds(n, 5, delta=2.5, standardizer=std)
    seen, compacted = set(), 0
    for k, rd in enumerate(rounds):
        # the flash attempt of the round, recomputed
        draft, _, _, _, res = ae.flash_batch(vc, rd["obs"], rd["ev"], rd["st"], rd["signs"], replan_size=4)
        # only the envs with a cached context and no forced refresh made an
        # attempt (compacted on the device); the others' words are -1
        use = (rd["hc0"] != 0) & (rd["fsr0"] < 2)
        assert torch.equal(res[use], rd["result"][use])
        assert (rd["result"][~use][:, :5] == -1).all() and (rd["branch"][~use] == -1).all()
        compacted += int(0 < int(use.sum()) <= 32)  # attempt gathered into the 32-env flash bucket
        path, planned, idx = _replan_ref(res.cpu().numpy(), rd["fsr0"].cpu().numpy(),
                                         rd["hc0"].cpu().numpy(), 2, 4)
        np.testing.assert_array_equal(rd["path"].cpu().numpy(), path)
        np.testing.assert_array_equal(rd["planned"].cpu().numpy(), planned)
        assert rd["nfb"] == len(idx)
        seen.update(path.tolist())
        acc = path == 0
        # accepted envs execute their draft
        assert torch.equal(rd["chunk"][torch.from_numpy(acc).cuda()], draft[torch.from_numpy(acc).cuda()])
        if len(idx):
            m = torch.from_numpy(idx.astype(np.int32)).cuda()
            full, status = ae.denoise_envs(m, rd["ed"][m.long()], rd["st"][m.long()], 10)
            assert (status[:, 0] == -1).all()
            torch.testing.assert_close(rd["chunk"][m.long()], full, rtol=2e-3,
                                       atol=2e-3 * full.abs().max().item())
        # switch_in_executed on the executed prefix of accepted rounds (runtime.py:321-323)
        ch = rd["chunk"].cpu().numpy()
        sg = rd["signs"].cpu().numpy()
        for e in range(n):
            want = bool(acc[e] and np.any(ch[e, :planned[e], -1] * sg[e] <= 0.0))
            assert bool(rd["sie"][e]) == want
        assert not rd["bad"].any()
        raw = rd["raw"].cpu().numpy()
        np.testing.assert_allclose(raw, ch * std.std.astype(np.float32) + std.mean.astype(np.float32),
                                   rtol=1e-6, atol=1e-6)
    # round 0 is a full round everywhere; later rounds mix flash and fallback paths
    assert (rounds[0]["path"] == 3).all()
    assert {0, 4}.issubset(seen) and ({1, 2} & seen)
    assert compacted >= 1


def test_replan_round_no_host_sync_and_launch_accounting():
    """The round is one graph launch: it enqueues without waiting for the GPU
    (the host returns while a long kernel still occupies the stream)."""
    import time

    import torch

    from paper_2605_13778_b200 import _capi

    n = 8
    ae, vc, rp, rounds = _run_rounds(n, 2, delta=2.5, standardizer=None)
    rd = rounds[-1]
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)  # ~0.1 s of GPU time ahead of the round
    t0 = time.perf_counter()
    c0 = _capi.launch_count()
    rp.round(rd["obs"], rd["ev"], rd["ed"], rd["st"], rd["signs"])
    dt = time.perf_counter() - t0
    assert _capi.launch_count() > c0
    torch.cuda.synchronize()
    assert dt < 0.05, f"round blocked the host for {dt * 1e3:.1f} ms"


def test_replan_round_full_only_and_single_env():
    """mode_flash = 0 (RuntimePolicy.mode == full_only): every round is a full
    round (path FULL, planned R) and the chunk is the Euler path; one env
    (bucket set {1}) goes through the same graph."""
    import torch

    from paper_2605_13778_b200 import _capi, pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    dcfg = pi0.AEConfig(**SMALL)
    for n in (1, 5):
        ae = pi0.ActionExpert(dcfg, seed=0, n_envs=n, kv_seed=1)
        vc = VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=2.5, gripper_window=6)
        rp = pi0.BatchedReplanner(ae, n, vc, replan_size=4, periodic_refresh=2, flash=False)
        g = torch.Generator(device="cuda").manual_seed(n)
        H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
        mk = lambda *sh: torch.randn(sh, generator=g, device="cuda")
        for _ in range(3):
            obs, ev, ed, st = mk(n, dcfg.draft_in), mk(n, H, D), mk(n, H, D), mk(n, S)
            chunk, path, planned, _, _ = rp.round(obs, ev, ed, st, torch.ones(n, device="cuda"))
            assert (path == _capi.SF_PATH_FULL).all() and (planned == 4).all()
            assert int(rp.n_fallback.item()) == n
            full, _ = ae.denoise_batch(ed, st, 10)
            torch.testing.assert_close(chunk, full, rtol=2e-3, atol=2e-3 * full.abs().max().item())


def test_replan_round_fp32_mode():
    """The replanning round in the fp32 mode (SF_AE_FP32): bookkeeping as
    run_episode, fallback chunks equal to the fp32-mode Euler of those envs."""
    import torch

    from paper_2605_13778_b200 import pi0
    from paper_2605_13778_b200.verifier import VerifierConfig

    dcfg = pi0.AEConfig(**SMALL)
    n = 6
    ae = pi0.ActionExpert(dcfg, seed=0, n_envs=n, kv_seed=1, draft_gripper_bias=6.0, precision="fp32")
    vc = VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=2.5, gripper_window=6)
    rp = pi0.BatchedReplanner(ae, n, vc, replan_size=4, periodic_refresh=2)
    g = torch.Generator(device="cuda").manual_seed(3)
    H, D, S = dcfg.horizon, dcfg.action_dim, dcfg.state_dim
    mk = lambda *sh: torch.randn(sh, generator=g, device="cuda")
    signs = torch.where(torch.arange(n, device="cuda") % 2 == 0, 1.0, -1.0)
    for r in range(3):
        obs, ev, ed, st = mk(n, dcfg.draft_in), mk(n, H, D), mk(n, H, D), mk(n, S)
        fsr0, hc0 = rp.fsr.cpu().numpy(), rp.has_cache.cpu().numpy()
        chunk, path, planned, _, result = rp.round(obs, ev, ed, st, signs)
        want_path, want_planned, idx = _replan_ref(result.cpu().numpy(), fsr0, hc0, 2, 4)
        np.testing.assert_array_equal(path.cpu().numpy(), want_path)
        np.testing.assert_array_equal(planned.cpu().numpy(), want_planned)
        if len(idx):
            m = torch.from_numpy(idx.astype(np.int32)).cuda()
            full, _ = ae.denoise_envs(m, ed[m.long()], st[m.long()], 10)
            torch.testing.assert_close(chunk[m.long()], full, rtol=1e-5, atol=1e-5 * full.abs().max().item())
