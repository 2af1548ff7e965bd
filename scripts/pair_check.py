"""pi0-scale verify outputs of the 1-SM persistent attention kernel
(SF_ATTN_SINGLE=1) vs the default 2-SM pair kernel on the same inputs.

usage: python scripts/pair_check.py
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2605_13778_b200.pi0 import PI0, ActionExpert
from paper_2605_13778_b200.verifier import VerifierConfig
E = 96
vc = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=0.15, gripper_window=24)
g = torch.Generator(device="cuda").manual_seed(0)
d = torch.randn((E, PI0.horizon, PI0.action_dim), generator=g, device="cuda")
e = torch.randn((E, PI0.horizon, PI0.action_dim), generator=g, device="cuda")
s = torch.randn((E, PI0.state_dim), generator=g, device="cuda")
outs = []
for flag in ("1", None):  # 1-SM kernel first, then the default 2-SM pair kernel
    if flag: os.environ["SF_ATTN_SINGLE"] = flag
    else: os.environ.pop("SF_ATTN_SINGLE", None)
    ae = ActionExpert(PI0, n_envs=E)
    outs.append([t.clone() for t in ae.verify_batch(vc, d, e, s)])
    del ae
for n, a, b in zip(["recon", "dist", "branch", "result"], *outs):
    if a.dtype.is_floating_point:
        print(n, "max|diff|", (a - b).abs().max().item(), "max|ref|", a.abs().max().item())
    else:
        print(n, "equal", bool(torch.equal(a, b)))
