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


_dev_cache: dict = {}


def device() -> torch.device:
    idx = torch._C._cuda_getDevice() if torch.cuda.is_initialized() else None
    d = _dev_cache.get(idx)
    if d is None:
        if not torch.cuda.is_available():
            raise RuntimeError("specflow_b200 requires a CUDA device (no CPU fallback)")
        idx = torch.cuda.current_device()
        d = _dev_cache[idx] = torch.device("cuda", idx)
    return d


def stream_ptr() -> int:
    """Raw handle of torch's current stream on the current device (the C-ABI
    launches there); ~0.1 us instead of ~3 us for current_stream()."""
    device()
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def to_dev(a, dtype: torch.dtype | None = None) -> torch.Tensor:
    """numpy/array-like -> contiguous device tensor in the current precision."""
    # a writable copy: reference arrays are often read-only (ActionChunk freezes its values)
    t = torch.as_tensor(np.array(a, dtype=np.float64, order="C"))
    return t.to(device=device(), dtype=dtype or tdtype(), non_blocking=False).contiguous()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class Staging:
    """Reusable pinned-host + device buffers for one call shape.

    Inputs are packed into ONE pinned host buffer and moved with ONE H2D copy;
    the kernel writes its values and int32 words into ONE device buffer that
    comes back with ONE D2H copy + stream synchronize (two ctypes calls, no
    torch copy / stream objects on the hot path), so a tiny round costs two
    copies and one launch.
    """

    _cache: dict = {}

    def __init__(self, n_in: int, n_out: int, n_words: int, dtype: torch.dtype):
        dev = device()
        self.dtype = dtype
        esz = torch.empty(0, dtype=dtype).element_size()
        self.esz = esz
        self.n_in, self.n_out, self.n_words = n_in, n_out, n_words
        self.words_off = (max(n_out, 1) * esz + 15) & ~15
        out_bytes = self.words_off + max(n_words, 1) * 4
        in_bytes = max(n_in, 1) * esz
        self.h_in = torch.empty(in_bytes, dtype=torch.uint8, pin_memory=True)
        self.d_in = torch.empty(in_bytes, dtype=torch.uint8, device=dev)
        self.h_out = torch.empty(out_bytes, dtype=torch.uint8, pin_memory=True)
        self.d_out = torch.empty(out_bytes, dtype=torch.uint8, device=dev)
        npdt = np.float32 if esz == 4 else np.float64
        self.h_in_np = self.h_in.numpy().view(npdt)
        ob = self.h_out.numpy()
        self.h_vals_np = ob[: max(n_out, 1) * esz].view(npdt)
        self.h_words_np = ob[self.words_off:].view(np.int32)
        self.d_in_ptr, self.h_in_ptr = self.d_in.data_ptr(), self.h_in.data_ptr()
        self.d_out_ptr, self.h_out_ptr = self.d_out.data_ptr(), self.h_out.data_ptr()
        self.extra: dict = {}  # per-shape ctypes argument structs built once by callers

    @classmethod
    def get(cls, key, n_in, n_out, n_words, dtype: torch.dtype | None = None) -> "Staging":
        dt = dtype or tdtype()
        k = (key, n_in, n_out, n_words, dt, torch._C._cuda_getDevice())
        st = cls._cache.get(k)
        if st is None:
            st = cls._cache[k] = Staging(n_in, n_out, n_words, dt)
        return st

    def upload(self, parts) -> list:
        """Pack host arrays into the pinned buffer, copy once; returns device
        pointers of each part (in order)."""
        hv = self.h_in_np
        ptrs, off = [], 0
        for p in parts:
            a = np.asarray(p, dtype=np.float64).ravel()
            hv[off: off + a.size] = a
            ptrs.append(self.d_in_ptr + off * self.esz)
            off += a.size
        _capi.check(_capi.lib().sf_copy_h2d(self.d_in_ptr, self.h_in_ptr, off * self.esz, stream_ptr()),
                    "staging upload")
        return ptrs

    def out_ptr(self, offset: int) -> int:
        return self.d_out_ptr + offset * self.esz

    def word_ptr(self, offset: int) -> int:
        return self.d_out_ptr + self.words_off + offset * 4

    def download(self, n_out: int, n_words: int):
        """Copy results back (syncs the stream); returns (values, words) numpy copies."""
        nbytes = self.words_off + n_words * 4 if n_words else n_out * self.esz
        _capi.check(_capi.lib().sf_copy_d2h_sync(self.h_out_ptr, self.d_out_ptr, nbytes, stream_ptr()),
                    "staging download")
        return (self.h_vals_np[:n_out].astype(np.float64), self.h_words_np[:n_words].copy())
