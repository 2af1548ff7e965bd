"""Batch-1 verify with the SF_TRACE build of the library (attention timeline
stamps printed by the first/last CTAs of each attention launch).

usage: SPECFLOW_B200_LIB=paper_2605_13778_b200/lib_trace/libspecflow_b200.so python scripts/attn_trace_b1.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_13778_b200.pi0 import PI0, ActionExpert
from paper_2605_13778_b200.verifier import VerifierConfig

cfg = PI0
vc = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=0.15, gripper_window=24)
g = torch.Generator(device="cuda").manual_seed(0)
d = torch.randn((1, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
e = torch.randn((1, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
s = torch.randn((1, cfg.state_dim), generator=g, device="cuda")
ae = ActionExpert(cfg, n_envs=1, flags=0)
for i in range(3):
    ae.verify_batch(vc, d, e, s)
    torch.cuda.synchronize()
    print("---- round", i, flush=True)
