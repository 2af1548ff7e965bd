"""Full-scale context refresh (Gemma-2B-style prefix encoder, P = 800) time
per prefill and achieved TFLOP/s: python scripts/prefill_bench.py --envs 1 4"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_13778_b200.pi0 import VLMConfig, VLMPrefill


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, nargs="+", default=[1, 4])
    args = ap.parse_args()
    cfg = VLMConfig()
    vlm = VLMPrefill(cfg)
    nq = cfg.q_heads * cfg.head_dim
    per_tok = 2 * cfg.layers * cfg.width * (nq + 2 * cfg.head_dim + nq + 3 * cfg.mlp)
    attn = 4 * cfg.layers * cfg.prefix_len * cfg.q_heads * cfg.head_dim  # per token (P keys)
    for E in args.envs:
        x = torch.randn((E, cfg.prefix_len, cfg.width), device="cuda")
        kp, vp = vlm.prefill(x)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            vlm.prefill(x, kp, vp)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / 5
        flops = E * cfg.prefix_len * (per_tok + attn)
        print(f"prefill envs={E}: {ms:.3f} ms  {flops / ms / 1e9:.0f} TFLOP/s  "
              f"({flops / 1e12:.2f} TFLOP)", flush=True)


if __name__ == "__main__":
    main()
