"""Drive pi0 verify / denoise graphs for profiling (ncu launch lists).

usage: python scripts/prof_pi0.py --envs 1 --mode verify --iters 2
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_13778_b200.pi0 import PI0, ActionExpert, SF_AE_GRAPH, SF_AE_PDL
from paper_2605_13778_b200.verifier import VerifierConfig


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=1)
    ap.add_argument("--mode", choices=["verify", "flash", "denoise"], default="verify")
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--eager", action="store_true")
    ap.add_argument("--nopdl", action="store_true")
    args = ap.parse_args()
    flags = (0 if args.eager else SF_AE_GRAPH) | (0 if args.nopdl else SF_AE_PDL)
    ae = ActionExpert(PI0, n_envs=args.envs, flags=flags)
    E, cfg = args.envs, PI0
    g = torch.Generator(device="cuda").manual_seed(0)
    obs = torch.randn((E, cfg.draft_in), generator=g, device="cuda")
    eps = torch.randn((E, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
    state = torch.randn((E, cfg.state_dim), generator=g, device="cuda")
    vcfg = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=0.15, gripper_window=24)
    draft = torch.randn((E, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
    for _ in range(args.iters):
        if args.mode == "verify":
            ae.verify_batch(vcfg, draft, eps, state)
        elif args.mode == "flash":
            ae.flash_batch(vcfg, obs, eps, state)
        else:
            ae.denoise_batch(draft, state, 10)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
