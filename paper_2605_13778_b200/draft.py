"""Draft model: single-pass chunk proposal on the device.

Mirrors ``specflow.draft`` (draft.py:29-61). ``propose`` runs the draft MLP on
the device; inside a speculative round (``runtime.flash_attempt``) the draft
forward is fused into the same launch as verification. Draft training
(draft.py:64-203) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _capi, _device
from .actions import STANDARDIZED, ActionChunk, ChannelLayout
from .flowpolicy import Observation
from .nets import Mlp


@dataclass
class DraftModel:
    """[world, task one-hot, robot state] -> H x D (draft.py:29-54)."""

    net: Mlp
    layout: ChannelLayout
    horizon: int
    n_tasks: int
    normalizer: object

    def __post_init__(self) -> None:
        if self.net.out_dim != self.horizon * self.layout.dim:
            raise ValueError("draft net output does not match horizon x dim")

    def features(self, obs: Observation) -> np.ndarray:
        if not 0 <= obs.task_id < self.n_tasks:
            raise ValueError(f"unknown task id {obs.task_id}")
        onehot = np.zeros(self.n_tasks)
        onehot[obs.task_id] = 1.0
        return np.concatenate([self.normalizer.norm_world(obs.world_features), onehot,
                               self.normalizer.norm_state(obs.robot_state)])


def propose(model: DraftModel, obs: Observation) -> ActionChunk:
    """One deterministic device forward (``sf_tiny_mlp_forward``), reshaped
    row-major to (H, D) (draft.py:57-61)."""
    feats = model.features(obs)
    hd = model.horizon * model.layout.dim
    stg = _device.Staging.get("propose", feats.size, hd, 1)
    (p_in,) = stg.upload([feats])
    _capi.check(_capi.lib().sf_tiny_mlp_forward(_device.code(), model.net.device().desc, p_in, 1,
                                                stg.out_ptr(0), _device.stream_ptr()), "propose")
    vals, _ = stg.download(hd, 0)
    return ActionChunk(values=vals.reshape(model.horizon, model.layout.dim), layout=model.layout,
                       space=STANDARDIZED)
