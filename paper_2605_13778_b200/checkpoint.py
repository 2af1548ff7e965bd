"""SFARRAYS checkpoint reader -> device-ready models.

Reads the reference's container (bench/checkpoint.py:24-83): 8-byte magic
``SFARRAYS``, little-endian u32 header length, JSON header (format version,
meta, per-array name/shape/dtype/offset/nbytes), raw little-endian payloads,
SHA-256 trailer over everything before it. The checksum and version are
verified before any array is materialised. Main/draft layouts follow
bench/checkpoint.py:118-199; weights are uploaded to the device lazily on
first use (``Mlp.device()``).
"""

from __future__ import annotations

import hashlib
import json
import struct
from pathlib import Path

import numpy as np

from .actions import ChannelLayout, Standardizer
from .draft import DraftModel
from .flowpolicy import ContextEncoder, ObsNormalizer, VelocityField
from .nets import Mlp

MAGIC = b"SFARRAYS"
FORMAT_VERSION = 1
_DTYPES = {"<f8": np.dtype("<f8"), "<i8": np.dtype("<i8")}


class CheckpointError(RuntimeError):
    pass


def load_arrays(path) -> tuple[dict, dict]:
    raw = Path(path).read_bytes()
    if len(raw) < len(MAGIC) + 4 + 32 or raw[: len(MAGIC)] != MAGIC:
        raise CheckpointError(f"{path}: not an SFARRAYS container")
    body, trailer = raw[:-32], raw[-32:]
    if hashlib.sha256(body).digest() != trailer:
        raise CheckpointError(f"{path}: checksum mismatch (truncated or corrupted)")
    (hlen,) = struct.unpack_from("<I", body, len(MAGIC))
    start = len(MAGIC) + 4
    header = json.loads(body[start: start + hlen].decode("utf-8"))
    if header.get("format_version") != FORMAT_VERSION:
        raise CheckpointError(f"{path}: unsupported format version {header.get('format_version')}")
    payload = memoryview(body)[start + hlen:]
    arrays = {}
    for e in header["arrays"]:
        dt = _DTYPES.get(e["dtype"])
        if dt is None:
            raise CheckpointError(f"{path}: unsupported dtype {e['dtype']}")
        lo, n = int(e["offset"]), int(e["nbytes"])
        if lo + n > len(payload):
            raise CheckpointError(f"{path}: array {e['name']} overruns the payload")
        arrays[e["name"]] = np.frombuffer(payload[lo: lo + n], dtype=dt).reshape(e["shape"]).copy()
    return arrays, header.get("meta", {})


def _mlp(prefix: str, n_layers: int, arrays: dict) -> Mlp:
    return Mlp(weights=[arrays[f"{prefix}.w{i}"] for i in range(n_layers)],
               biases=[arrays[f"{prefix}.b{i}"] for i in range(n_layers)])


def _normalizer(arrays: dict) -> ObsNormalizer:
    return ObsNormalizer(arrays["norm.world_mean"], arrays["norm.world_std"],
                         arrays["norm.state_mean"], arrays["norm.state_std"])


def load_main_checkpoint(path):
    """-> (ContextEncoder, VelocityField, Standardizer, meta) (bench/checkpoint.py:147-175)."""
    arrays, meta = load_arrays(path)
    if meta.get("kind") != "main":
        raise CheckpointError(f"{path}: expected a main-policy checkpoint")
    layout = ChannelLayout(**meta["layout"])
    enc = ContextEncoder(net=_mlp("encoder", meta["encoder_layers"], arrays),
                         n_tasks=meta["n_tasks"], normalizer=_normalizer(arrays))
    field = VelocityField(net=_mlp("field", meta["field_layers"], arrays), horizon=meta["horizon"],
                          dim=layout.dim, emb_dim=meta["emb_dim"], state_dim=meta["state_dim"],
                          layout=layout)
    return enc, field, Standardizer(mean=arrays["std.mean"], std=arrays["std.std"]), meta


def load_draft_checkpoint(path):
    """-> (DraftModel, meta) (bench/checkpoint.py:189-199)."""
    arrays, meta = load_arrays(path)
    if meta.get("kind") != "draft":
        raise CheckpointError(f"{path}: expected a draft checkpoint")
    model = DraftModel(net=_mlp("draft", meta["draft_layers"], arrays),
                       layout=ChannelLayout(**meta["layout"]), horizon=meta["horizon"],
                       n_tasks=meta["n_tasks"], normalizer=_normalizer(arrays))
    return model, meta
