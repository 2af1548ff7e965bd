"""tcgen05 GEMM (csrc/gemm.cuh) against a torch fp32 reference on the same
bf16-rounded operands: both orientations, split-K, odd shapes, RMS row scale."""

import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _run(M, N, K, bn, splits, swap, kind=0, ssq=None):
    import torch

    from paper_2605_13778_b200 import _capi

    torch.manual_seed(M * 7 + N * 13 + K + bn + splits)
    x = torch.randn(M, K, device="cuda").bfloat16()  # token rows
    w = (torch.randn(N, K, device="cuda") * 0.05).bfloat16()  # feature rows (weights)
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if kind == 0 else torch.bfloat16)
    a, ra, b, rb = (w, N, x, M) if swap else (x, M, w, N)
    ssq_ptr, groups = (None, 0) if ssq is None else (ssq.data_ptr(), ssq.shape[0])
    rc = _capi.lib().sf_dbg_gemm(a.data_ptr(), ra, b.data_ptr(), rb, K, bn, splits, int(swap), kind,
                                 out.data_ptr(), N, M, N, ssq_ptr, groups, M, 1.0 / K,
                                 torch.cuda.current_stream().cuda_stream)
    _capi.check(rc, "gemm")
    ref = x.float() @ w.float().T
    if ssq is not None:
        ref = ref * torch.rsqrt(ssq.sum(0) / K + 1e-6)[:, None]
    return out.float(), ref


@pytest.mark.parametrize("M,N,K,bn,splits", [
    (128, 256, 64, 256, 1),
    (256, 512, 1024, 256, 1),
    (200, 300, 512, 128, 1),
    (1000, 512, 2048, 256, 4),
    (64, 64, 128, 64, 2),
])
def test_normal_orientation(M, N, K, bn, splits):
    import torch

    out, ref = _run(M, N, K, bn, splits, swap=False)
    torch.testing.assert_close(out, ref, rtol=2e-3, atol=2e-3)


@pytest.mark.parametrize("M,N,K,bn,splits", [
    (208, 2560, 1024, 208, 0),   # qkv at batch 1, K=4 (auto split-K)
    (208, 1024, 2048, 208, 0),   # o-proj
    (208, 1024, 4096, 208, 16),  # down-proj
    (51, 8192, 1024, 64, 0),     # Euler step rows
    (416, 1024, 1024, 208, 3),   # bn smaller than rows -> 2 token tiles
    (17, 300, 192, 32, 1),
])
def test_swap_ab_split_k(M, N, K, bn, splits):
    import torch

    out, ref = _run(M, N, K, bn, splits, swap=True)
    torch.testing.assert_close(out, ref, rtol=2e-3, atol=2e-3)


def test_split_k_is_deterministic():
    import torch

    a, _ = _run(208, 1024, 4096, 208, 16, swap=True)
    b, _ = _run(208, 1024, 4096, 208, 16, swap=True)
    assert torch.equal(a, b)


@pytest.mark.parametrize("swap", [False, True])
def test_rms_row_scale_and_bf16_store(swap):
    import torch

    M, N, K = 208, 512, 1024
    ssq = torch.rand(8, M, device="cuda") * 100 + 1
    out, ref = _run(M, N, K, 208 if swap else 256, 0 if swap else 1, swap, kind=1, ssq=ssq)
    torch.testing.assert_close(out, ref, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("M,N,K", [
    (1024, 512, 1024),
    (1500, 768, 2048),   # ragged last row tile; 3 feature tiles (odd pair count)
    (4096, 2560, 1024),  # qkv-shaped; more tiles than CTA pairs
])
def test_pair_kernel(M, N, K):
    """Batched shapes (bn = 256, >= 1024 rows) run on 2-SM CTA pairs
    (tcgen05.mma.cta_group::2, gemm_pair_kernel)."""
    import torch

    out, ref = _run(M, N, K, 256, 1, swap=False)
    torch.testing.assert_close(out, ref, rtol=2e-3, atol=2e-3)


def test_pair_kernel_rms_bf16():
    import torch

    M, N, K = 2048, 1024, 1024
    ssq = torch.rand(8, M, device="cuda") * 100 + 1
    out, ref = _run(M, N, K, 256, 1, False, kind=1, ssq=ssq)
    torch.testing.assert_close(out, ref, rtol=1e-2, atol=1e-2)
