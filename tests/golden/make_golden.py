"""Generate golden vectors by running the REAL reference (``specflow``).

Run in the build container only (``/root/reference`` does not exist on the GPU
box); the outputs are committed under ``tests/golden/``:

* ``cfg1_tiny.npz``   — cfg1 (D=7, H=50, K=3) random-init models, several
  seeded rounds: draft, reconstructed endpoints, distances, branch prefixes,
  gripper switch, full-round Euler chunk, context embedding. Weights are NOT
  stored: they are regenerated from the recorded seeds with ``init_mlp``
  (nets.py:47-57) and pinned by per-layer checksums stored here.
* ``cfg2_main.ckpt`` / ``cfg2_draft.ckpt`` — the reference's own trained
  default models (``specflow run --seed 7``), SFARRAYS format
  (bench/checkpoint.py:24-83).
* ``cfg2_trace.npz``  — every flash_attempt / full_round the reference made
  while running the seed-7 episode plus 12 ``episode_seed_for_trial(0, t)``
  episodes: inputs (draft features, cache embedding, normalized state, sign,
  seeds) and outputs (draft, distances, branch prefixes, switch, Euler chunk),
  plus each round's path/planned record from ``run_episode``.

Usage:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py \
            --models-dir /tmp/cfg2/models
"""

from __future__ import annotations

import argparse
import shutil
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from specflow import nets, runtime  # noqa: E402
from specflow.actions import STANDARDIZED, ActionChunk, ChannelLayout  # noqa: E402
from specflow.draft import DraftModel, propose  # noqa: E402
from specflow.flowpolicy import (  # noqa: E402
    ConditioningCache,
    ContextEncoder,
    DenoiseConfig,
    ObsNormalizer,
    Observation,
    VelocityField,
    encode_context,
    integrate_flow,
)
from specflow.verifier import VerifierConfig, verify  # noqa: E402


def _checksum(a):
    a = np.asarray(a, np.float64)
    return np.array([a.sum(), (a * a).sum(), a.ravel()[0], a.ravel()[-1]])


def make_cfg1(out: Path) -> None:
    """cfg1: ChannelLayout(3,3), H=50, K=3, tau=(0.25,0.5,0.75)."""
    layout = ChannelLayout(3, 3)
    h, d = 50, layout.dim
    world_dim, n_tasks, state_dim = 5, 2, 3
    emb_in = world_dim + n_tasks
    rec = {"layout": np.array([3, 3]), "h": h}
    model_seed = 1234
    rng = np.random.default_rng(model_seed)
    enc_net = nets.init_mlp([emb_in, 64, 32], rng)
    field_net = nets.init_mlp([h * d + 1 + emb_in + 32 + state_dim, 256, 256, h * d], rng)
    draft_net = nets.init_mlp([world_dim + n_tasks + state_dim, 160, 160, h * d], rng)
    rec["model_seed"] = model_seed
    for name, net in (("enc", enc_net), ("field", field_net), ("draft", draft_net)):
        rec[f"{name}_sizes"] = np.array(net.sizes)
        rec[f"{name}_checksums"] = np.stack([_checksum(w) for w in net.weights])
    norm = ObsNormalizer.identity(world_dim, state_dim)
    encoder = ContextEncoder(net=enc_net, n_tasks=n_tasks, normalizer=norm)
    field = VelocityField(net=field_net, horizon=h, dim=d, emb_dim=encoder.embed_dim,
                          state_dim=state_dim, layout=layout)
    draft = DraftModel(net=draft_net, layout=layout, horizon=h, n_tasks=n_tasks, normalizer=norm)

    taus = (0.25, 0.5, 0.75)
    cases = []
    case_rng = np.random.default_rng(99)
    n_cases = 12
    for c in range(n_cases):
        obs = Observation(world_features=case_rng.normal(size=world_dim),
                          task_id=int(case_rng.integers(0, n_tasks)),
                          robot_state=case_rng.normal(size=state_dim))
        cache = encode_context(encoder, obs)
        state = norm.norm_state(obs.robot_state)
        dchunk = propose(draft, obs)
        sign = -1.0 if c % 2 == 0 else 1.0
        if c % 3 == 1:
            # draft gripper one-signed on the current side (the gate can then
            # only fire from a reconstructed branch)
            vals = dchunk.values.copy()
            vals[:, -1] = sign * (np.abs(vals[:, -1]) + 0.1)
            dchunk = ActionChunk(values=vals, layout=layout, space=STANDARDIZED)
        metric = "linf" if c % 4 == 3 else "l2"
        window = None if c % 2 == 0 else 24
        delta = [0.15, 0.96, 1.42, 1.83][c % 4]
        vseed = runtime._stream_seed(1000 + c, c, 1)
        cfg = VerifierConfig(timesteps=taus, delta=delta, metric=metric, gripper_window=window)
        rep = verify(field, dchunk, cache, state, cfg, np.random.default_rng(vseed),
                     current_gripper_sign=sign, noise_seed=vseed)
        dseed = runtime._stream_seed(1000 + c, c, 0)
        full = integrate_flow(field, cache, state, DenoiseConfig(10), np.random.default_rng(dseed))
        cases.append(dict(
            world=obs.world_features, task=obs.task_id, robot_state=obs.robot_state,
            emb=cache.embedding, state=state, draft=dchunk.values, sign=sign,
            metric=0 if metric == "l2" else 1, window=-1 if window is None else window,
            delta=delta, vseed=vseed, dseed=dseed, recon=rep.reconstructed,
            distances=rep.distances, branch=np.array(rep.branch_prefixes), prefix=rep.prefix,
            switch=rep.gripper_switch_detected, full=full,
            eps=np.random.default_rng(vseed).standard_normal((h, d)),
        ))
    for key in cases[0]:
        rec[f"case_{key}"] = np.stack([np.asarray(cs[key]) for cs in cases])
    rec["taus"] = np.array(taus)
    np.savez_compressed(out / "cfg1_tiny.npz", **rec)
    print(f"cfg1: {n_cases} cases -> {out / 'cfg1_tiny.npz'}")


def make_cfg2(out: Path, models_dir: Path, n_trials: int) -> None:
    from specflow.bench import checkpoint as ckpt
    from specflow.bench.config import DEFAULT_CONFIG
    from specflow.bench import harness

    shutil.copy(models_dir / "main.ckpt", out / "cfg2_main.ckpt")
    shutil.copy(models_dir / "draft.ckpt", out / "cfg2_draft.ckpt")
    encoder, field, standardizer, _ = ckpt.load_main_checkpoint(models_dir / "main.ckpt")
    draft_model, _ = ckpt.load_draft_checkpoint(models_dir / "draft.ckpt")
    models = runtime.Models(encoder=encoder, field=field, standardizer=standardizer, draft=draft_model)
    config = DEFAULT_CONFIG

    calls = []  # one entry per flash_attempt / full_round
    orig_flash, orig_full = runtime.flash_attempt, runtime.full_round
    current = {"episode": -1}

    def flash_wrap(obs, models_, policy, state, round_index, episode_seed):
        draft_chunk, report, seed = orig_flash(obs, models_, policy, state, round_index, episode_seed)
        calls.append(dict(
            kind=1, episode=current["episode"], round=round_index, seed=seed,
            dfeat=draft_model.features(obs), efeat=encoder.features(obs),
            emb=state.cache.embedding,
            state=models_.norm_state(obs.robot_state), sign=state.gripper_sign,
            draft=draft_chunk.values, distances=report.distances,
            branch=np.array(report.branch_prefixes), prefix=report.prefix,
            switch=report.gripper_switch_detected, chunk=np.zeros_like(draft_chunk.values),
            raw_grip=obs.robot_state[2],
        ))
        return draft_chunk, report, seed

    def full_wrap(obs, models_, policy, round_index, tick, episode_seed):
        chunk, cache, seed = orig_full(obs, models_, policy, round_index, tick, episode_seed)
        h = chunk.values.shape[0]
        calls.append(dict(
            kind=0, episode=current["episode"], round=round_index, seed=seed,
            dfeat=draft_model.features(obs), efeat=encoder.features(obs),
            emb=cache.embedding,
            state=models_.norm_state(obs.robot_state), sign=0.0,
            draft=np.zeros_like(chunk.values), distances=np.zeros((2, h)),
            branch=np.zeros(2, dtype=int), prefix=0, switch=False, chunk=chunk.values,
            raw_grip=obs.robot_state[2],
        ))
        return chunk, cache, seed

    runtime.flash_attempt, runtime.full_round = flash_wrap, full_wrap
    rounds = []
    try:
        seeds = [7] + [harness.episode_seed_for_trial(0, t) for t in range(n_trials)]
        for ep, seed in enumerate(seeds):
            current["episode"] = ep
            _, records = harness.run_single_episode(config, models, seed, "demo", "large")
            for r in records:
                rounds.append(dict(
                    episode=ep, round=r.index, path=r.path, planned=r.planned,
                    prefix=-1 if r.prefix is None else r.prefix,
                    switch=-1 if r.gripper_switch is None else int(r.gripper_switch),
                ))
    finally:
        runtime.flash_attempt, runtime.full_round = orig_flash, orig_full

    rec = {"episode_seeds": np.array(seeds, dtype=np.int64)}
    for key in calls[0]:
        rec[f"call_{key}"] = np.stack([np.asarray(c[key]) for c in calls])
    paths = sorted({r["path"] for r in rounds})
    rec["path_names"] = np.array(paths)
    for key in ("episode", "round", "planned", "prefix", "switch"):
        rec[f"round_{key}"] = np.array([r[key] for r in rounds], dtype=np.int64)
    rec["round_path"] = np.array([paths.index(r["path"]) for r in rounds], dtype=np.int64)
    ver = config["verifier"]
    rec["taus"] = np.array(ver["timesteps"], dtype=np.float64)
    rec["delta"] = float(ver["delta"])
    rec["window"] = int(ver["gripper_window"])
    rec["replan_size"] = int(config["chunk"]["replan_size"])
    rec["num_steps"] = int(config["denoise"]["num_steps"])
    np.savez_compressed(out / "cfg2_trace.npz", **rec)
    n_flash = int(sum(c["kind"] for c in calls))
    print(f"cfg2: {len(seeds)} episodes, {len(rounds)} rounds, {n_flash} verify calls, "
          f"{len(calls) - n_flash} full rounds, paths={paths}")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--models-dir", type=Path, default=Path("/tmp/cfg2/models"))
    ap.add_argument("--trials", type=int, default=12)
    ap.add_argument("--skip-cfg2", action="store_true")
    args = ap.parse_args()
    make_cfg1(HERE)
    if not args.skip_cfg2:
        make_cfg2(HERE, args.models_dir, args.trials)


if __name__ == "__main__":
    main()
