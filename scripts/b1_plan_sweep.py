"""In-graph sweep of the batch-1 verify GEMM plans (GPU).

The static plan rule (csrc/pi0.cu, "batch-1 plan tuning") picks a token tile
(bn) and a K-split count (S) per layer GEMM class (qkv, o, gate/up, down) for
the K-branch verify (204 token rows at cfg3). SF_TUNE's serialised per-GEMM
timings are quantised to ~2.07 us steps (kernel completion polling without
PDL), so this script instead times the WHOLE speculative round (draft +
verify graph with PDL, `ActionExpert.flash_batch`) for each candidate, one
class at a time (coordinate descent from the rule's plan), through the
SF_B1_PLAN override. Prints the best "bn:S,..." string.

python scripts/b1_plan_sweep.py [--passes 2]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13778_b200 import pi0  # noqa: E402
from paper_2605_13778_b200.verifier import VerifierConfig  # noqa: E402

TAUS = (0.2, 0.4, 0.6, 0.8)
CANDS = {
    0: [(b, s) for b in (208, 112, 64) for s in (1, 2, 3, 4, 6)],   # qkv  N=2560 K=1024
    1: [(b, s) for b in (208, 112, 64) for s in (2, 3, 4, 6, 8)],   # o    N=1024 K=2048
    2: [(b, s) for b in (208, 112, 64) for s in (1, 2)],            # gu   N=8192 K=1024
    3: [(b, s) for b in (208, 112, 64) for s in (2, 3, 4, 6, 8)],   # down N=1024 K=4096
}
TILES_A = {0: 20, 1: 8, 2: 64, 3: 8}


def p50(fn, iters=40):
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def measure(plan, inputs):
    if plan is None:
        os.environ.pop("SF_B1_PLAN", None)
    else:
        os.environ["SF_B1_PLAN"] = ",".join(f"{b}:{s}" for b, s in plan)
    obs, eps, state, signs = inputs
    ae = pi0.ActionExpert(pi0.PI0, seed=0, n_envs=1, kv_seed=1)
    vcfg = VerifierConfig(timesteps=TAUS, delta=5.64, gripper_window=24)
    out = ae.flash_batch(vcfg, obs, eps, state, signs)
    for _ in range(5):
        ae.flash_batch(vcfg, obs, eps, state, signs, outputs=out)
    torch.cuda.synchronize()
    t = p50(lambda: ae.flash_batch(vcfg, obs, eps, state, signs, outputs=out))
    res = out[0].clone()
    del ae
    torch.cuda.synchronize()
    return t, res


def main():
    passes = int(sys.argv[sys.argv.index("--passes") + 1]) if "--passes" in sys.argv else 2
    rng = np.random.default_rng(5)
    dev = "cuda"
    obs = torch.from_numpy(rng.standard_normal((1, 64)).astype(np.float32)).to(dev)
    eps = torch.from_numpy(rng.standard_normal((1, 50, 32)).astype(np.float32)).to(dev)
    state = torch.from_numpy(rng.standard_normal((1, 32)).astype(np.float32)).to(dev)
    signs = torch.ones(1, device=dev)
    inputs = (obs, eps, state, signs)
    t_rule, _ = measure(None, inputs)
    print(f"rule plan: spec round p50 {t_rule:.4f} ms", flush=True)
    plan = [(0, 0)] * 4
    best_t = measure(plan, inputs)[0]
    for ps in range(passes):
        for cls in range(4):
            for cand in CANDS[cls]:
                b, s = cand
                if TILES_A[cls] * ((204 + b - 1) // b) * s > 2 * 148:
                    continue
                trial = list(plan)
                trial[cls] = cand
                try:
                    t, _ = measure(trial, inputs)
                except Exception as e:  # a plan that does not fit (SMEM, splits)
                    print(f"  pass {ps} cls {cls} {cand}: failed ({e})", flush=True)
                    continue
                print(f"  pass {ps} cls {cls} bn={b} S={s}: {t:.4f} ms", flush=True)
                if t < best_t * 0.995:
                    best_t, plan = t, trial
            print(f"pass {ps} cls {cls}: best so far {plan} {best_t:.4f} ms", flush=True)
    s = ",".join(f"{b}:{s}" for b, s in plan)
    print(f"BEST SF_B1_PLAN={s} spec round p50 {best_t:.4f} ms (rule {t_rule:.4f} ms)")


if __name__ == "__main__":
    main()
