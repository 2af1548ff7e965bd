"""Batch-1 layer-stack megakernel vs the per-op kernel chain: same inputs,
compare verify outputs and time both (graph + PDL).

usage: python scripts/stack_check.py
"""

import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_13778_b200.pi0 import PI0, ActionExpert
from paper_2605_13778_b200.verifier import VerifierConfig


def p50(fn, n=30):
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def run(no_stack):
    if no_stack:
        os.environ.pop("SF_STACK", None)
    else:
        os.environ["SF_STACK"] = "1"
    cfg = PI0
    vc = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=0.15, gripper_window=24)
    g = torch.Generator(device="cuda").manual_seed(0)
    d = torch.randn((1, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
    e = torch.randn((1, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
    s = torch.randn((1, cfg.state_dim), generator=g, device="cuda")
    ae = ActionExpert(cfg, n_envs=1)
    out = ae.verify_batch(vc, d, e, s)
    torch.cuda.synchronize()
    res = [t.clone() for t in out]
    for _ in range(3):
        ae.verify_batch(vc, d, e, s, outputs=out)
    t_verify = p50(lambda: ae.verify_batch(vc, d, e, s, outputs=out))
    # Euler full path (10 steps)
    start = torch.randn((1, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
    full, _ = ae.denoise_batch(start, s, 10)
    torch.cuda.synchronize()
    t_full = p50(lambda: ae.denoise_batch(start, s, 10), n=10)
    return res, full.clone(), t_verify, t_full


def main():
    ref, full_ref, tv0, tf0 = run(True)
    print(f"per-op chain : verify p50 {tv0:.3f} ms, 10-step full {tf0:.3f} ms", flush=True)
    got, full_got, tv1, tf1 = run(False)
    print(f"megakernel   : verify p50 {tv1:.3f} ms, 10-step full {tf1:.3f} ms", flush=True)
    names = ["recon", "dist", "branch", "result"]
    for n, a, b in zip(names, ref, got):
        if a.dtype.is_floating_point:
            err = (a - b).abs().max().item()
            scale = a.abs().max().item()
            print(f"  {n:7s}: max |diff| {err:.3e} (max |ref| {scale:.3e})")
        else:
            print(f"  {n:7s}: equal={bool(torch.equal(a, b))}")
    err = (full_ref - full_got).abs().max().item()
    print(f"  full   : max |diff| {err:.3e} (max |ref| {full_ref.abs().max().item():.3e})")


if __name__ == "__main__":
    main()
