"""Warm per-kernel device times of one eager pi0 verify round (sf_ae_profile_verify).

usage: python scripts/kernel_times.py --envs 1
"""

import argparse
import ctypes
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_13778_b200 import _capi
from paper_2605_13778_b200.pi0 import PI0, ActionExpert
from paper_2605_13778_b200.verifier import VerifierConfig, make_cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, nargs="+", default=[1])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--per-layer", action="store_true")
    args = ap.parse_args()
    cfg = PI0
    ae = ActionExpert(cfg, n_envs=max(args.envs))
    vc = make_cfg(VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=0.15, gripper_window=24), -1.0)
    names = ["embed"] + [f"L{l}.{n}" for l in range(cfg.layers) for n in ("qkv", "attn", "o", "gu", "down")] + [
        "head", "verify_epi"]
    for E in args.envs:
        g = torch.Generator(device="cuda").manual_seed(0)
        d = torch.randn((E, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
        e = torch.randn((E, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
        s = torch.randn((E, cfg.state_dim), generator=g, device="cuda")
        buf = (ctypes.c_float * 256)()
        n = ctypes.c_int()
        best = None
        for _ in range(args.reps):
            _capi.check(_capi.lib().sf_ae_profile_verify(
                ae._h, E, ctypes.byref(vc), d.data_ptr(), e.data_ptr(), s.data_ptr(), buf, 256,
                ctypes.byref(n), torch.cuda.current_stream().cuda_stream), "profile")
            t = list(buf[: n.value])
            best = t if best is None else [min(a, b) for a, b in zip(best, t)]
        agg = defaultdict(list)
        for name, t in zip(names, best):
            agg[name.split(".")[-1]].append(t)
        total = sum(best)
        print(f"envs={E}: {len(best)} kernels, {total:.1f} us total (eager, warm, no PDL)")
        if args.per_layer:
            print("  attn per layer:", " ".join(f"{t:.0f}" for t in agg["attn"]))
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            print(f"  {k:10s} n={len(v):3d} sum {sum(v):9.1f} us ({100 * sum(v) / total:4.1f}%)  "
                  f"avg {sum(v) / len(v):8.2f} us  min {min(v):7.2f}  max {max(v):7.2f}")


if __name__ == "__main__":
    main()
