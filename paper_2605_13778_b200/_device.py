"""Device plumbing: precision selection, streams, host<->device staging.

PyTorch is used only for device memory and streams; all arithmetic on the
path runs in the library's own sm_100a kernels.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _capi

_state = threading.local()

PRECISIONS = {"fp32": (_capi.SF_F32, torch.float32, np.float32),
              "fp64": (_capi.SF_F64, torch.float64, np.float64)}


def get_precision() -> str:
    return getattr(_state, "precision", "fp64")


def set_precision(name: str) -> None:
    """fp64 (default, the reference's arithmetic) or fp32 (north-star fp32 mode)."""
    if name not in PRECISIONS:
        raise ValueError(f"unknown precision {name!r}")
    _state.precision = name


class precision:
    """Context manager: ``with precision("fp32"): ...``."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        self.prev = get_precision()
        set_precision(self.name)

    def __exit__(self, *exc):
        set_precision(self.prev)


def code() -> int:
    return PRECISIONS[get_precision()][0]


def tdtype() -> torch.dtype:
    return PRECISIONS[get_precision()][1]


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("specflow_b200 requires a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def to_dev(a, dtype: torch.dtype | None = None) -> torch.Tensor:
    """numpy/array-like -> contiguous device tensor in the current precision."""
    t = torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
    return t.to(device=device(), dtype=dtype or tdtype(), non_blocking=False).contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class Staging:
    """Reusable pinned-host + device buffers for one call shape.

    Inputs are packed into ONE pinned host vector and moved with ONE H2D copy;
    outputs are written by the kernel into ONE device vector (plus an int32
    word vector) and read back with ONE D2H copy each, so a tiny round costs
    two copies and one launch.
    """

    _cache: dict = {}

    def __init__(self, n_in: int, n_out: int, n_words: int, dtype: torch.dtype):
        dev = device()
        self.dtype = dtype
        self.h_in = torch.empty(max(n_in, 1), dtype=dtype, pin_memory=True)
        self.d_in = torch.empty(max(n_in, 1), dtype=dtype, device=dev)
        self.d_out = torch.empty(max(n_out, 1), dtype=dtype, device=dev)
        self.h_out = torch.empty(max(n_out, 1), dtype=dtype, pin_memory=True)
        self.d_words = torch.empty(max(n_words, 1), dtype=torch.int32, device=dev)
        self.h_words = torch.empty(max(n_words, 1), dtype=torch.int32, pin_memory=True)

    @classmethod
    def get(cls, key, n_in, n_out, n_words) -> "Staging":
        dt = tdtype()
        k = (key, n_in, n_out, n_words, dt, torch.cuda.current_device())
        st = cls._cache.get(k)
        if st is None:
            st = cls._cache[k] = Staging(n_in, n_out, n_words, dt)
        return st

    def upload(self, parts) -> list:
        """Pack host arrays into the pinned buffer, copy once; returns device
        pointers of each part (in order)."""
        hv = self.h_in.numpy()
        ptrs, off = [], 0
        esz = self.d_in.element_size()
        for p in parts:
            a = np.asarray(p, dtype=np.float64).ravel()
            hv[off: off + a.size] = a
            ptrs.append(self.d_in.data_ptr() + off * esz)
            off += a.size
        self.d_in[:off].copy_(self.h_in[:off], non_blocking=True)
        return ptrs

    def out_ptr(self, offset: int) -> int:
        return self.d_out.data_ptr() + offset * self.d_out.element_size()

    def word_ptr(self, offset: int) -> int:
        return self.d_words.data_ptr() + offset * 4

    def download(self, n_out: int, n_words: int):
        """Copy results back (syncs the stream); returns (values, words) numpy views."""
        if n_out:
            self.h_out[:n_out].copy_(self.d_out[:n_out], non_blocking=True)
        self.h_words[:n_words].copy_(self.d_words[:n_words], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return (self.h_out[:n_out].numpy().astype(np.float64), self.h_words[:n_words].numpy().copy())
