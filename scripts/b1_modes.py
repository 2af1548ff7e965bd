"""Batch-1 verify latency under eager / graph / graph+PDL launch modes."""

import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_13778_b200.pi0 import PI0, SF_AE_GRAPH, SF_AE_PDL, ActionExpert
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


def main():
    cfg = PI0
    vc = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=0.15, gripper_window=24)
    g = torch.Generator(device="cuda").manual_seed(0)
    d = torch.randn((1, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
    e = torch.randn((1, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
    s = torch.randn((1, cfg.state_dim), generator=g, device="cuda")
    ae = ActionExpert(cfg, n_envs=1)
    for name, flags in (("eager", 0), ("eager+pdl", SF_AE_PDL), ("graph", SF_AE_GRAPH),
                        ("graph+pdl", SF_AE_GRAPH | SF_AE_PDL)):
        ae.flags = flags
        out = ae.verify_batch(vc, d, e, s)
        for _ in range(3):
            ae.verify_batch(vc, d, e, s, outputs=out)
        torch.cuda.synchronize()
        print(f"{name:10s}: verify p50 {p50(lambda: ae.verify_batch(vc, d, e, s, outputs=out)):.3f} ms")


if __name__ == "__main__":
    main()
