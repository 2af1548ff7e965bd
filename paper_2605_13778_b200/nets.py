"""Tanh MLP container (nets.py:16-57) and its device-resident form.

Only the inference half of the reference's ``nets`` is on the hot path; the
reference's backward/AdamW (nets.py:116-211) are training and out of scope.
Weights keep the reference layout ``(n_out, n_in)`` so the kernels stream
each output neuron's row contiguously.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _capi, _device


@dataclass
class Mlp:
    """Fully connected net: tanh hidden layers, identity output (nets.py:16-44)."""

    weights: list
    biases: list
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self) -> None:
        if not self.weights or len(self.weights) != len(self.biases):
            raise ValueError("weights and biases must be non-empty and matching")
        prev = None
        for i, (w, b) in enumerate(zip(self.weights, self.biases)):
            w = np.asarray(w, dtype=np.float64)
            b = np.asarray(b, dtype=np.float64)
            if w.ndim != 2 or b.shape != (w.shape[0],):
                raise ValueError(f"layer {i} has inconsistent shapes")
            if prev is not None and w.shape[1] != prev:
                raise ValueError(f"layer {i} input does not match layer {i - 1} output")
            if not (np.isfinite(w).all() and np.isfinite(b).all()):
                raise ValueError(f"layer {i} has non-finite parameters")
            prev = w.shape[0]
        if len(self.weights) > _capi.SF_MAX_LAYERS:
            raise ValueError(f"at most {_capi.SF_MAX_LAYERS} layers are supported on device")

    @property
    def sizes(self) -> tuple:
        return (int(np.shape(self.weights[0])[1]),) + tuple(int(np.shape(w)[0]) for w in self.weights)

    @property
    def in_dim(self) -> int:
        return self.sizes[0]

    @property
    def out_dim(self) -> int:
        return self.sizes[-1]

    def invalidate_device(self) -> None:
        """Drop device copies (call after mutating weights in place)."""
        self._device.clear()

    def device(self) -> "DeviceMlp":
        key = _device.get_precision()
        dm = self._device.get(key)
        if dm is None:
            dm = DeviceMlp(self)
            self._device[key] = dm
        return dm


class DeviceMlp:
    """Weights uploaded once in the current precision + the C-ABI descriptor."""

    def __init__(self, net: Mlp):
        self.tensors = []
        self.desc = _capi.SfMlp()
        self.desc.n_layers = len(net.weights)
        for i, s in enumerate(net.sizes):
            self.desc.sizes[i] = s
        dt = _device.tdtype()
        pad = 16 // torch.empty(0, dtype=dt).element_size()
        for i, (w, b) in enumerate(zip(net.weights, net.biases)):
            w = np.asarray(w, dtype=np.float64)
            ld = -(-w.shape[1] // pad) * pad  # rows padded to 16 B for TMA bulk staging
            wp = np.zeros((w.shape[0], ld))
            wp[:, : w.shape[1]] = w
            tw, tb = _device.to_dev(wp), _device.to_dev(b)
            self.tensors += [tw, tb]
            self.desc.ld[i] = ld
            self.desc.w[i] = tw.data_ptr()
            self.desc.b[i] = tb.data_ptr()


def init_mlp(sizes, rng: np.random.Generator) -> Mlp:
    """Xavier-normal weights, zero biases, same rng call order (nets.py:47-57)."""
    sizes = [int(s) for s in sizes]
    if len(sizes) < 2:
        raise ValueError("need at least input and output sizes")
    ws, bs = [], []
    for fan_in, fan_out in zip(sizes, sizes[1:]):
        ws.append(rng.normal(0.0, np.sqrt(2.0 / (fan_in + fan_out)), size=(fan_out, fan_in)))
        bs.append(np.zeros(fan_out))
    return Mlp(weights=ws, biases=bs)


def n_params(net: Mlp) -> int:
    return int(sum(np.size(w) + np.size(b) for w, b in zip(net.weights, net.biases)))


def flop_count(net: Mlp) -> int:
    """Multiply-add = 2 FLOPs, plus bias and activation (nets.py:73-79)."""
    return int(sum(2 * w.shape[0] * w.shape[1] + 2 * w.shape[0] for w in map(np.asarray, net.weights)))

