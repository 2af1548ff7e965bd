"""Shared builders for the tiny-model tests (cfg1 random-init, cfg2 trained)."""

from __future__ import annotations

import numpy as np

from conftest import GOLDEN


def cfg1_golden():
    return dict(np.load(GOLDEN / "cfg1_tiny.npz"))


def cfg1_numpy_weights(g):
    """Regenerate cfg1 weights exactly as make_golden.py drew them (init_mlp
    order: encoder, field, draft from one generator)."""
    from oracle import specflow_oracle as so

    rng = np.random.default_rng(int(g["model_seed"]))
    enc = so.init_mlp(list(g["enc_sizes"]), rng)
    field = so.init_mlp(list(g["field_sizes"]), rng)
    draft = so.init_mlp(list(g["draft_sizes"]), rng)
    return enc, field, draft


def cfg1_device_models(g):
    """Product-side model objects with the same weights (regenerated with the
    product's own init_mlp, which follows nets.py:47-57)."""
    from paper_2605_13778_b200.actions import ChannelLayout
    from paper_2605_13778_b200.draft import DraftModel
    from paper_2605_13778_b200.flowpolicy import ContextEncoder, ObsNormalizer, VelocityField
    from paper_2605_13778_b200.nets import init_mlp

    rng = np.random.default_rng(int(g["model_seed"]))
    enc_net = init_mlp(list(g["enc_sizes"]), rng)
    field_net = init_mlp(list(g["field_sizes"]), rng)
    draft_net = init_mlp(list(g["draft_sizes"]), rng)
    layout = ChannelLayout(*[int(x) for x in g["layout"]])
    h = int(g["h"])
    world_dim, n_tasks, state_dim = 5, 2, 3
    norm = ObsNormalizer.identity(world_dim, state_dim)
    enc = ContextEncoder(net=enc_net, n_tasks=n_tasks, normalizer=norm)
    field = VelocityField(net=field_net, horizon=h, dim=layout.dim, emb_dim=enc.embed_dim,
                          state_dim=state_dim, layout=layout)
    draft = DraftModel(net=draft_net, layout=layout, horizon=h, n_tasks=n_tasks, normalizer=norm)
    return enc, field, draft, layout


def cfg2_trace():
    return dict(np.load(GOLDEN / "cfg2_trace.npz"))


def cfg2_models():
    from paper_2605_13778_b200 import checkpoint as ck

    enc, field, std, _ = ck.load_main_checkpoint(GOLDEN / "cfg2_main.ckpt")
    draft, _ = ck.load_draft_checkpoint(GOLDEN / "cfg2_draft.ckpt")
    return enc, field, std, draft
