"""ctypes binding of the C-ABI in ``include/specflow_b200.h``.

The shared library is built in-tree (``paper_2605_13778_b200/lib``) by
``__graft_entry__.build()``. There is no CPU fallback: importing a device entry
point without the library raises immediately.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libspecflow_b200.so"

SF_OK, SF_EINVAL, SF_ENONFINITE, SF_ERUNTIME, SF_ECUDA = 0, 1, 2, 3, 4
SF_F32, SF_F64 = 0, 1
SF_MAX_LAYERS = 8
SF_MAX_K = 16
TINY_MAX_K = 8  # branch rows of one fused tiny-field launch (csrc/tiny.cu kMaxRows)
SF_METRIC = {"l2": 0, "linf": 1}
SF_RESULT_WORDS = 8
RES_PREFIX, RES_SWITCH, RES_PATH, RES_PLANNED, RES_NONFINITE = 0, 1, 2, 3, 4
# specflow_b200.h: SF_PATH_* device path codes, SF_RES_* result word indices
SF_PATH_FLASH_ACCEPTED, SF_PATH_FLASH_REJECTED, SF_PATH_FLASH_PHASE = 0, 1, 2
SF_PATH_FULL, SF_PATH_PERIODIC = 3, 4
SF_RES_PREFIX, SF_RES_SWITCH, SF_RES_PATH, SF_RES_PLANNED, SF_RES_NONFINITE = 0, 1, 2, 3, 4
PATH_CODES = ("flash_accepted", "flash_rejected_fallback", "flash_phase_fallback")


class SfMlp(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int),
        ("sizes", ctypes.c_int * (SF_MAX_LAYERS + 1)),
        ("ld", ctypes.c_int * SF_MAX_LAYERS),
        ("w", ctypes.c_void_p * SF_MAX_LAYERS),
        ("b", ctypes.c_void_p * SF_MAX_LAYERS),
    ]


class SfVerifyCfg(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_int),
        ("taus", ctypes.c_double * SF_MAX_K),
        ("delta", ctypes.c_double),
        ("metric", ctypes.c_int),
        ("window", ctypes.c_int),
        ("current_sign", ctypes.c_double),
        ("phase_fallback", ctypes.c_int),
        ("prefix_cap", ctypes.c_int),
        ("replan_size", ctypes.c_int),
    ]


class SfVerifyOut(ctypes.Structure):
    _fields_ = [
        ("draft", ctypes.c_void_p),
        ("reconstructed", ctypes.c_void_p),
        ("distances", ctypes.c_void_p),
        ("branch_prefixes", ctypes.c_void_p),
        ("result", ctypes.c_void_p),
    ]


class SfReplanPolicy(ctypes.Structure):
    _fields_ = [("mode_flash", ctypes.c_int), ("periodic_refresh", ctypes.c_int),
                ("num_steps", ctypes.c_int), ("std_mean", ctypes.c_void_p), ("std_std", ctypes.c_void_p)]


class SfReplanOut(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("chunk", "chunk_raw", "path", "planned",
                                               "switch_in_executed", "nonfinite", "branch_prefixes",
                                               "result", "n_fallback")]


_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double

# name -> (restype, argtypes); every name here is declared in include/specflow_b200.h
SIGNATURES = {
    "sf_last_error": (ctypes.c_char_p, []),
    "sf_version": (_I, []),
    "sf_launch_count": (ctypes.c_int64, [_I]),
    "sf_copy_h2d": (_I, [_P, _P, ctypes.c_size_t, _P]),
    "sf_copy_d2h_sync": (_I, [_P, _P, ctypes.c_size_t, _P]),
    "sf_tiny_flash_round": (_I, [_I, ctypes.POINTER(SfMlp), _P, ctypes.POINTER(SfMlp), _P, _I, _P, _I,
                                 _P, _I, _I, _I, ctypes.POINTER(SfVerifyCfg),
                                 ctypes.POINTER(SfVerifyOut), _P]),
    "sf_tiny_full_round": (_I, [_I, ctypes.POINTER(SfMlp), _P, _I, ctypes.POINTER(SfMlp), _P, _I, _P,
                                _I, _I, _I, _P, _P, _P, _P]),
    "sf_tiny_mlp_forward": (_I, [_I, ctypes.POINTER(SfMlp), _P, _I, _P, _P]),
    "sf_tiny_field_eval": (_I, [_I, ctypes.POINTER(SfMlp), _P, _P, _I, _P, _I, _P, _I, _I, _I, _P,
                                _P, _P]),
    "sf_interpolate": (_I, [_I, _P, _P, _P, _I, _I, _P, _P]),
    "sf_verify_epilogue": (_I, [_I, _P, _P, _P, _I, _I, _I, ctypes.POINTER(SfVerifyCfg),
                                ctypes.POINTER(SfVerifyOut), _P]),
    "sf_prefix_length": (_I, [_I, _P, _I, _I, _D, _P, _P]),
    "sf_continuous_distances": (_I, [_I, _P, _P, _I, _I, _I, _I, _P, _P]),
    "sf_gripper_switch": (_I, [_I, _P, _I, _I, _I, _D, _I, _P, _P]),
    "sf_euler_update": (_I, [_I, _P, _P, _I, _I, _I, _P, _P]),
    # include/specflow_b200_pi0.h
    "sf_ae_create": (_I, [_P, _P, _P]),
    "sf_ae_destroy": (_I, [_P]),
    "sf_ae_set_prefix": (_I, [_P, _P, _P, _I]),
    "sf_ae_refresh_prefix": (_I, [_P, _P]),
    "sf_ae_verify": (_I, [_P, _I, ctypes.POINTER(SfVerifyCfg), _P, _P, _P, _P,
                          ctypes.POINTER(SfVerifyOut), _I, _P]),
    "sf_ae_denoise": (_I, [_P, _I, _I, _P, _P, _P, _P, _I, _P]),
    "sf_ae_denoise_envs": (_I, [_P, _I, _P, _I, _P, _P, _P, _P, _I, _P]),
    "sf_replan_update": (_I, [_I, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P]),
    "sf_vlm_create": (_I, [_P, _P, _P]),
    "sf_vlm_destroy": (_I, [_P]),
    "sf_vlm_prefill": (_I, [_P, _I, _P, _P, _P, _P]),
    "sf_ae_flash_round": (_I, [_P, _I, ctypes.POINTER(SfVerifyCfg), _P, _P, _P, _P,
                               ctypes.POINTER(SfVerifyOut), _I, _P]),
    "sf_ae_time_op": (_I, [_P, _I, _I, _I, _I, _P]),
    "sf_ae_profile_verify": (_I, [_P, _I, ctypes.POINTER(SfVerifyCfg), _P, _P, _P, _P, _I, _P, _P]),
    "sf_ae_velocity": (_I, [_P, _I, _I, _P, _P, _P, _P, _P]),
    "sf_ae_replan_round": (_I, [_P, _I, ctypes.POINTER(SfVerifyCfg), ctypes.POINTER(SfReplanPolicy), _P, _P,
                                _P, _P, _P, _P, _P, ctypes.POINTER(SfReplanOut), _I, _P]),
    "sf_ae_replan_kernels": (_I, [_P, _P]),
    "sf_fill_hash_uniform": (_I, [_P, _I, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_double, _P]),
    # include/specflow_b200_internal.h (kernel unit-test hooks)
    "sf_dbg_gemm": (_I, [_P, _I, _P, _I, _I, _I, _I, _I, _I, _P, _I, _I, _I, _P, _I, _I,
                         ctypes.c_float, _P]),
    "sf_dbg_gemm_time": (_I, [_P, _I, _P, _I, _I, _I, _I, _I, _P, _I, _I, _P, _P]),
    "sf_dbg_gemm_trace": (_I, [_P, _I, _P, _I, _I, _I, _I, _P, _P, _P]),
    "sf_ae_b1_trace": (_I, [_P, _P, ctypes.c_size_t]),
    "sf_tiny_trace": (_I, [_I, _P]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load the library once; fail loudly if it is missing (no CPU fallback)."""
    global _lib
    if _lib is None:
        path = os.environ.get("SPECFLOW_B200_LIB", str(_LIB_PATH))
        if not Path(path).exists():
            raise LibraryMissing(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        handle = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int, what: str = "") -> None:
    """Map C-ABI status codes to the reference's exception types."""
    if rc == SF_OK:
        return
    msg = lib().sf_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == SF_EINVAL:
        raise ValueError(msg)
    if rc == SF_ENONFINITE:
        raise FloatingPointError(msg)
    raise RuntimeError(msg)


def host_doubles(vals):
    """HOST double array for the C-ABI's `const double*` host arguments."""
    return (ctypes.c_double * len(vals))(*[float(v) for v in vals])


def launch_count(reset: bool = False) -> int:
    return int(lib().sf_launch_count(1 if reset else 0))
