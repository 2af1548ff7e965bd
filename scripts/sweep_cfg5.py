"""cfg5 (BASELINE.json configs[4]): sweep K in {1, 2, 4, 8}, chunk H in {16,
50, 100} and the acceptance threshold delta, on the pi0-scale Action Expert
(random init, bf16) at batch 1 (latency) and over a batch of envs (accepted
prefix length and fallback rate vs delta).

tau_k = k / (K + 1) (generalising verifier.py:33). Random-init drafts are far
from the field's reconstructions, so the delta grid is taken at quantiles of
the observed per-step distances. Gripper drafts are made
one-signed so the phase gate does not mask the threshold sweep; phase
fallbacks are still counted.

usage: python scripts/sweep_cfg5.py [--envs 64] [--out profiles/r1/cfg5_sweep.json]
"""

import argparse
import dataclasses
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

from paper_2605_13778_b200 import _capi
from paper_2605_13778_b200.pi0 import PI0, ActionExpert
from paper_2605_13778_b200.verifier import VerifierConfig


def p50(fn, n=20):
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=64)
    ap.add_argument("--out", default="profiles/r1/cfg5_sweep.json")
    args = ap.parse_args()
    rows = []
    for H in (16, 50, 100):
        cfg = dataclasses.replace(PI0, horizon=H)
        E = args.envs
        ae = ActionExpert(cfg, n_envs=E)
        g = torch.Generator(device="cuda").manual_seed(H)
        D, S, F = cfg.action_dim, cfg.state_dim, cfg.draft_in
        obs = torch.randn((E, F), generator=g, device="cuda")
        eps = torch.randn((E, H, D), generator=g, device="cuda")
        state = torch.randn((E, S), generator=g, device="cuda")
        draft = torch.randn((E, H, D), generator=g, device="cuda")
        draft[..., -1] = draft[..., -1].abs() + 0.1  # one-signed gripper: g * sign > 0, no switch in the draft
        signs = torch.ones(E, device="cuda")
        for K in (1, 2, 4, 8):
            taus = tuple((k + 1) / (K + 1) for k in range(K))
            vc = VerifierConfig(timesteps=taus, delta=0.15, gripper_window=24)
            # batch-1 latency (graph + PDL)
            o1 = ae.flash_batch(vc, obs[:1], eps[:1], state[:1], signs[:1])
            v1 = ae.verify_batch(vc, draft[:1], eps[:1], state[:1], signs[:1])
            for _ in range(3):
                ae.flash_batch(vc, obs[:1], eps[:1], state[:1], signs[:1], outputs=o1)
                ae.verify_batch(vc, draft[:1], eps[:1], state[:1], signs[:1], outputs=v1)
            torch.cuda.synchronize()
            spec = p50(lambda: ae.flash_batch(vc, obs[:1], eps[:1], state[:1], signs[:1], outputs=o1))
            ver = p50(lambda: ae.verify_batch(vc, draft[:1], eps[:1], state[:1], signs[:1], outputs=v1))
            # delta sweep over E envs: thresholds at distance quantiles
            _, dist, _, _ = ae.verify_batch(vc, draft, eps, state, signs)
            d = dist.float().cpu().numpy()
            qs = (0.0, 0.1, 0.25, 0.5, 0.75, 0.9)
            sweep = []
            for q in qs:
                delta = float(np.quantile(d, q)) if q > 0 else 0.0
                vcd = VerifierConfig(timesteps=taus, delta=delta, gripper_window=24)
                _, _, branch, result = ae.verify_batch(vcd, draft, eps, state, signs)
                r = result.cpu().numpy()
                L = r[:, _capi.SF_RES_PREFIX]
                path = r[:, _capi.SF_RES_PATH]
                sweep.append({"distance_quantile": q, "delta": delta, "mean_prefix": float(L.mean()),
                              "accept_rate": float((path == _capi.SF_PATH_FLASH_ACCEPTED).mean()),
                              "rejected_rate": float((path == _capi.SF_PATH_FLASH_REJECTED).mean()),
                              "phase_fallback_rate": float((path == _capi.SF_PATH_FLASH_PHASE).mean())})
            row = {"H": H, "K": K, "taus": list(taus), "spec_round_b1_ms": spec, "verify_b1_ms": ver,
                   "envs": E, "delta_sweep": sweep}
            rows.append(row)
            print(json.dumps({k: row[k] for k in ("H", "K", "spec_round_b1_ms", "verify_b1_ms")}),
                  [round(x["mean_prefix"], 1) for x in sweep], flush=True)
        del ae
        torch.cuda.empty_cache()
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(json.dumps({"workload": "cfg5 sweep (pi0-scale AE, random init, bf16, 1 GPU)",
                               "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
