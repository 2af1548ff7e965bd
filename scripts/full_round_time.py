"""p50 of the cfg3 10-step Euler full round and the batch-1 verify (graph+PDL)."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

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


cfg = PI0
ae = ActionExpert(cfg, n_envs=1)
g = torch.Generator(device="cuda").manual_seed(0)
d = torch.randn((1, cfg.horizon, cfg.action_dim), generator=g, device="cuda")
s = torch.randn((1, cfg.state_dim), generator=g, device="cuda")
vc = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=0.15, gripper_window=24)
out = ae.verify_batch(vc, d, d, s)
for _ in range(3):
    ae.denoise_batch(d, s, 10)
    ae.verify_batch(vc, d, d, s, outputs=out)
torch.cuda.synchronize()
print(f"full {p50(lambda: ae.denoise_batch(d, s, 10)):.3f} ms  verify {p50(lambda: ae.verify_batch(vc, d, d, s, outputs=out), 40):.3f} ms")
