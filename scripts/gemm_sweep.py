"""Sweep GEMM configurations with sf_dbg_gemm_time (device time per launch)."""

import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_13778_b200 import _capi


def t(M, N, K, bn, splits, swap, pdl=0, iters=50):
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = (torch.randn(N, K, device="cuda") * 0.05).bfloat16()
    out = torch.empty(M, N, device="cuda")
    a, ra, b, rb = (w, N, x, M) if swap else (x, M, w, N)
    us = ctypes.c_float()
    _capi.check(_capi.lib().sf_dbg_gemm_time(a.data_ptr(), ra, b.data_ptr(), rb, K, bn, splits,
                                             int(swap), out.data_ptr(), iters, pdl, ctypes.byref(us),
                                             torch.cuda.current_stream().cuda_stream), "time")
    wbytes = N * K * 2
    flops = 2.0 * M * N * K
    print(f"M={M:6d} N={N:5d} K={K:5d} bn={bn:3d} S={splits:2d} swap={int(swap)} pdl={pdl}: "
          f"{us.value:8.2f} us  {wbytes / us.value / 1e3:7.1f} GB/s(w)  {flops / us.value / 1e6:7.1f} TF/s")


def main():
    t(16, 128, 64, 16, 1, True)
    t(208, 128, 64, 208, 1, True)
    for s in (1, 2, 4, 8, 16):
        t(208, 1024, 4096, 208, s, True)
    for s in (1, 2, 4, 8):
        t(208, 1024, 4096, 208, s, True, pdl=1)
    for s in (1, 2, 4):
        t(208, 8192, 1024, 208, s, True)
    t(208, 2560, 1024, 208, 6, True)
    t(13312, 8192, 1024, 256, 1, False)
    t(13312, 2560, 1024, 256, 1, False)
    t(13312, 1024, 4096, 256, 1, False)
    t(106496, 8192, 1024, 256, 1, False, iters=5)


if __name__ == "__main__":
    main()


def trace(M, N, K, bn, splits):
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = (torch.randn(N, K, device="cuda") * 0.05).bfloat16()
    out = torch.empty(M, N, device="cuda")
    st = (ctypes.c_ulonglong * 12)()
    _capi.check(_capi.lib().sf_dbg_gemm_trace(w.data_ptr(), N, x.data_ptr(), M, K, bn, splits,
                                              out.data_ptr(), st,
                                              torch.cuda.current_stream().cuda_stream), "trace")
    t0 = st[0]
    names = ["entry", "prologue", "producer_done", "mma_committed", "rs_ready", "acc_ready",
             "staged", "csync1", "reduced", "csync2", "epi_end", "tmem_freed"]
    print(f"trace M={M} N={N} K={K} S={splits}: " +
          " ".join(f"{n}={(v - t0) / 1e3:.2f}" if v else f"{n}=-" for n, v in zip(names, st)))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "trace":
    trace(208, 1024, 4096, 208, 8)
    trace(208, 8192, 1024, 208, 2)
    trace(208, 2560, 1024, 208, 6)
    trace(16, 128, 64, 16, 1)


def sweep(M):
    """Batch-1 shape sweep: token tile (bn) x K splits for the four layer GEMMs."""
    shapes = {"qkv": (2560, 1024), "o": (1024, 2048), "gu": (8192, 1024), "down": (1024, 4096)}
    for name, (N, K) in shapes.items():
        best = None
        for bn in sorted({((M + 15) // 16) * 16, ((M + 31) // 32) * 16, ((M + 63) // 64) * 16, 32, 16}, reverse=True):
            tiles = ((N + 127) // 128) * ((M + bn - 1) // bn)
            for S in (1, 2, 3, 4, 6, 8, 12, 16):
                if tiles * S > 160 or S > K // 64:
                    continue
                x = torch.randn(M, K, device="cuda").bfloat16()
                w = (torch.randn(N, K, device="cuda") * 0.05).bfloat16()
                out = torch.empty(M, N, device="cuda")
                us = ctypes.c_float()
                _capi.check(_capi.lib().sf_dbg_gemm_time(w.data_ptr(), N, x.data_ptr(), M, K, bn, S, 1,
                                                         out.data_ptr(), 30, 1, ctypes.byref(us),
                                                         torch.cuda.current_stream().cuda_stream), "time")
                print(f"{name} M={M} bn={bn:3d} S={S:2d} ctas={tiles * S:3d}: {us.value:7.2f} us")
                if best is None or us.value < best[0]:
                    best = (us.value, bn, S)
        print(f"BEST {name} M={M}: {best[0]:.2f} us bn={best[1]} S={best[2]}", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "sweep":
    for M in (208, 64):
        sweep(M)
