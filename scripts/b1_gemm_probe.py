"""Batch-1 swap-AB GEMM probe: per-phase %globaltimer stamps of CTA (0,0,0)
and back-to-back (PDL) device time per launch for the cfg3 verify shapes
(208 token rows) over a range of split-K counts.

usage: python scripts/b1_gemm_probe.py [--rows 208]
"""

import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_13778_b200 import _capi

SHAPES = {"qkv": (2560, 1024), "o": (1024, 2048), "gu": (8192, 1024), "down": (1024, 4096)}
NAMES = ["entry", "prologue", "prod_issued", "mma_commit", "rs_ready", "acc_ready", "partial",
         "csync", "reduce_epi", "csync2", "epi_end", "tmem_free"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=208)
    args = ap.parse_args()
    lib = _capi.lib()
    s = torch.cuda.current_stream().cuda_stream
    M = args.rows
    for name, (N, K) in SHAPES.items():
        A = (torch.randn((N, K), device="cuda") * 0.02).to(torch.bfloat16)
        B = torch.randn((M, K), device="cuda").to(torch.bfloat16)
        out = torch.empty((M, N), device="cuda")
        for splits in (1, 2, 3, 4, 6, 8, 12, 16):
            if (K // 64) < splits:
                continue
            us = ctypes.c_float()
            rc_t = lib.sf_dbg_gemm_time(A.data_ptr(), N, B.data_ptr(), M, K, M, splits, 1, out.data_ptr(),
                                        50, 1, ctypes.byref(us), s)
            us_np = ctypes.c_float()
            lib.sf_dbg_gemm_time(A.data_ptr(), N, B.data_ptr(), M, K, M, splits, 1, out.data_ptr(),
                                 50, 0, ctypes.byref(us_np), s)
            st = (ctypes.c_ulonglong * 16)()
            rc = lib.sf_dbg_gemm_trace(A.data_ptr(), N, B.data_ptr(), M, K, M, splits, out.data_ptr(), st, s)
            if rc or rc_t:
                print(f"{name} S={splits}: rc {rc}/{rc_t} {lib.sf_last_error().decode()}")
                continue
            t0 = st[0]
            marks = " ".join(f"{NAMES[i]}={(st[i] - t0) / 1e3:.2f}" for i in range(1, 12) if st[i])
            gbs = 2 * N * K / (us.value * 1e-6) / 1e9
            print(f"{name:5s} N={N} K={K} S={splits:2d}: pdl {us.value:6.2f} us ({gbs:6.0f} GB/s)  "
                  f"nopdl {us_np.value:6.2f} us | {marks}")


if __name__ == "__main__":
    main()
