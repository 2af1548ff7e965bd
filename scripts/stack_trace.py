"""One eager batch-1 verify through the megakernel with SF_STACK_TRACE=1."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["SF_STACK_TRACE"] = "1"
os.environ["SF_STACK"] = "1"

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
for i in range(2):
    ae.verify_batch(vc, d, e, s)
    torch.cuda.synchronize()
