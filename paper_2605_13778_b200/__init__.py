"""B200-native (sm_100a) speculative-replanning path of Realtime-VLA FLASH.

Drop-in for the reference ``specflow`` hot path (draft -> K-timestep parallel
verify -> longest-consistent-prefix accept -> phase-aware fallback gate; the
Euler full path on fallback). Host code mirrors the reference API; all
arithmetic runs in hand-written CUDA kernels behind the C-ABI in
``include/specflow_b200.h`` (``lib/libspecflow_b200.so``). No CPU fallback.
"""

from ._device import get_precision, precision, set_precision  # noqa: F401

__version__ = "0.1.0"
