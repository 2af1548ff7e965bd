#!/usr/bin/env python
"""Benchmark of the B200-native speculative-replanning path (driver contract).

Headline workload (BASELINE.json configs[3], "cfg4"): the pi0-scale Action
Expert (18 layers, width 1024, 8x256 MQA heads, GeGLU 4096; ~314M params,
bf16) over a per-env random-init VLM prefix KV cache (800 tokens), chunk
50 x 32, K = 4 verification timesteps; 512 synthetic environments sharded
contiguously across the GPUs (no collective on the hot path).

One step = one REPLANNING ROUND for every env (run_episode's round,
runtime.py:238-326, minus the conveyor): the batched speculative attempt
(draft MLP -> 4-branch verify -> longest consistent prefix -> gripper gate ->
decision, one CUDA graph), the device round bookkeeping (periodic refresh
PF = 2, prefix cap R = 12, fallback compaction), then the 10-step Euler full
path for the envs that fell back (full / periodic / rejected / phase).

Workload (per env, seeded by ``sharding.env_seed(SEED, env)`` so it does not
depend on the GPU count): obs, verify / denoise noise, state; the draft holds
a one-signed gripper column (draft output bias +20 on the gripper channel) and
odd envs run with the opposite current gripper sign, so half the envs take
the phase fallback; delta = DELTA_CFG4 sits at the median of the deciding
distance of the other half, so accepted and rejected rounds both occur.

value       = replanning rounds / s over all GPUs (device time, max over ranks)
value_spec  = speculative attempts / s (the flash graph alone)
e2e         = replanning rounds / s through BatchedReplanner.round with HOST
              inputs: pinned H2D of obs / noise / state / signs and D2H of the
              chunk to execute + path + planned every step
parity      = after the timed region, a sample of envs re-verified by the
              oracle (decisions vs the bf16-mirroring oracle, endpoints vs the
              unrounded fp32 model)
latency_b1  = cfg3 batch-1 p50 (spec round, verify, 10-step full round) and
              the reference-facing plugin calls (numpy in / numpy out)
latency_tiny= cfg1 p50 of runtime.flash_attempt / full_round next to the
              reference algorithm's CPU p50 in the same run
roofline    = dominant kernel (gate/up GEMM, tensor-bound) + batch-1 verify (HBM)
cpu_baseline / --impl reference = the CPU oracle port of the reference path
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "p50 speculative-round & full-round latency (ms); rounds/sec at 1/2/4/8 B200"
SEED = 0
TAUS = (0.2, 0.4, 0.6, 0.8)
WINDOW = 24
GRIP = 20.0          # draft gripper-column output bias (one-signed drafts)
REPLAN = 12          # replan_size R (config.py default)
PF = 2               # periodic refresh
# Median over the even (same-sign) envs of the deciding distance
# max_k d[k, 0] of the 512-env workload (bench.py --calibrate; the value is
# re-checked every run: line["decision_mix"]["delta_quantile"]).
DELTA_CFG4 = 5.64


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--envs", type=int, default=512, help="total environments (all GPUs)")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-audit", action="store_true")
    ap.add_argument("--audit-envs", type=int, default=8)
    ap.add_argument("--cpu-sample-envs", type=int, default=2)
    ap.add_argument("--calibrate", action="store_true", help="print deciding-distance quantiles and exit")
    ap.add_argument("--sweep", action="store_true", help="cfg5 sweep (K, H, delta) instead of the bench line")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo: shard + seed + gather plumbing only (no GPU, no kernels)")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def respawn(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run
    with one rank per GPU (the driver's own launch line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(ROOT / "bench.py")] + sys.argv[1:]
    return subprocess.call(cmd)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d["bf16_tflops_sustained"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", ",".join(str(g) for g in self.gpus)],
                stdout=self.file, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        self.file.flush()
        rows = []
        for line in Path(self.file.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((int(parts[1]), int(parts[2]), float(parts[3]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [r for r in rows if r[2] > 200.0] or rows
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "power_w_max": max(r[2] for r in rows), "samples": len(loaded), "reasons": reasons}


def event_ms(fn, iters, stream=None):
    import torch

    s = stream or torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(iters):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / iters


def p50_ms(fn, iters):
    import torch

    times = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b))
    return statistics.median(times)


def host_p50_ms(fn, iters):
    times = []
    for _ in range(iters):
        t0 = time.perf_counter()
        fn()
        times.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(times)


# --------------------------------------------------------------- workload

def env_inputs(env: int, H=50, D=32, S=32, F=64):
    """Per-env round inputs from SeedSequence([SEED, env]) (harness.py:435-436
    style): independent of how envs are sharded across GPUs."""
    import numpy as np

    from paper_2605_13778_b200.sharding import env_seed

    rng = np.random.default_rng(env_seed(SEED, env))
    obs = rng.standard_normal(F).astype(np.float32)
    eps_v = rng.standard_normal((H, D)).astype(np.float32)
    eps_d = rng.standard_normal((H, D)).astype(np.float32)
    state = rng.standard_normal(S).astype(np.float32)
    sign = 1.0 if env % 2 == 0 else -1.0
    return obs, eps_v, eps_d, state, sign


def shard_inputs(lo: int, hi: int):
    import numpy as np

    cols = list(zip(*[env_inputs(e) for e in range(lo, hi)]))
    return [np.stack(c).astype(np.float32) for c in cols[:4]] + [np.array(cols[4], np.float32)]


# --------------------------------------------------------------- CPU side

def cpu_replan_round(env: int, cfg=None, w=None, dw=None, delta=DELTA_CFG4):
    """One replanning round of env `env` on the host with the reference's
    algorithm: the draft (propose, draft.py:57-61), verify (verifier.py:109-150,
    oracle/specflow_oracle.verify driving the numpy pi0 field), the decision
    (runtime.py:286-320) and, on fallback, the 10-step Euler full path
    (flowpolicy.py:273-292). Returns (path, seconds)."""
    import numpy as np

    from oracle import pi0_oracle as po
    from oracle import specflow_oracle as so

    cfg = cfg or po.AEConfig()
    w = w if w is not None else po.make_weights(cfg, 0)
    dw = dw if dw is not None else po.make_draft_weights(cfg, 0)
    kv = po.make_prefix_kv(cfg, 1, env)
    obs, eps_v, eps_d, state, sign = env_inputs(env)
    t0 = time.perf_counter()
    draft = po.draft_forward(cfg, dw, obs[None])[0].astype(np.float64)
    draft[:, -1] += GRIP
    vel = lambda x, t: po.field_velocity(cfg, w, kv, [(x.astype(np.float32), t)], state)[0]
    rep = so.verify(vel, draft, eps_v.astype(np.float64), TAUS, delta, cfg.action_dim - 1, "l2", WINDOW,
                    sign)
    path, _ = so.fallback_decision(rep["prefix"], rep["gripper_switch_detected"], cfg.horizon,
                                   replan_size=REPLAN)
    if path != so.PATH_FLASH_ACCEPTED:
        so.integrate_flow(vel, eps_d.astype(np.float64), 10)
    return path, time.perf_counter() - t0


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host cores, one env
    replanning round per step (alternating a same-sign and an opposite-sign
    env, so flash-only and fallback rounds both enter the mean)."""
    if rank != 0:
        return
    from oracle import pi0_oracle as po

    cfg = po.AEConfig()
    w, dw = po.make_weights(cfg, 0), po.make_draft_weights(cfg, 0)
    cores = os.cpu_count() or 1
    times, paths = [], []
    for i in range(args.warmup + args.steps):
        path, dt = cpu_replan_round(i % args.envs, cfg, w, dw)
        if i >= args.warmup:
            times.append(dt)
            paths.append(path)
    per = statistics.mean(times)
    value = 1.0 / per
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rounds/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "cfg4 replanning round per env (pi0-scale AE, K=4, H=50, D=32, P=800; "
                               "draft + verify + decision + fallback Euler)",
                   "envs_total": args.envs, "delta": DELTA_CFG4, "paths": {p: paths.count(p) for p in set(paths)}},
        "cpu_baseline": {"value": value, "unit": "rounds/s", "cores": cores, "kind": "port",
                         "sample": "1 env replanning round per step (numpy oracle: reference verify / "
                                   "decision / integrate_flow driving the pi0 field), envs alternate sign"},
        "e2e": {"value": value, "unit": "rounds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- dry run (CPU / gloo)

def run_dry(args, rank, world):
    """Multi-rank plumbing on the CPU: contiguous shards, N-independent per-env
    seeds, the after-timing gathers. Prints one JSON line from rank 0."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_13778_b200.sharding import gather_counts, max_over_ranks, shard_range

    if world > 1:
        dist.init_process_group("gloo")
    lo, hi = shard_range(args.envs, rank, world)
    obs, eps_v, eps_d, state, signs = shard_inputs(lo, hi)
    # an N-independent checksum of the shard's inputs and a per-rank "time"
    chk = torch.tensor([float(np.float64(obs).sum() + np.float64(eps_v).sum() + np.float64(state).sum())],
                       dtype=torch.float64)
    counts = torch.tensor([int((signs > 0).sum()), 0, int((signs < 0).sum())], dtype=torch.int64)
    shards = torch.tensor([lo, hi], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(chk)
        got = [torch.empty_like(shards) for _ in range(world)]
        dist.all_gather(got, shards)
        shards_all = [g.tolist() for g in got]
    else:
        shards_all = [shards.tolist()]
    counts = gather_counts(counts).tolist()
    ms = max_over_ranks(float(rank + 1))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "envs_total": args.envs, "shards": shards_all,
                          "input_checksum": float(chk.item()), "sign_counts": counts,
                          "max_over_ranks": ms}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------- GPU side

def audit(ae, vcfg, lo, draft, recon, dist, branch, result, eps_v, state, signs, envs_local, dev,
          round_chunk=None, round_path=None, eps_d=None):
    """Re-verify sampled envs with the oracle after the timed region: device
    draft vs the oracle draft; decisions vs the bf16-mirroring oracle (flips
    counted with their distance to delta, |d - delta| < 1e-4 reported as
    near-threshold); endpoints vs the unrounded fp32 model; and the executed
    chunk of (up to 2) sampled envs that fell back in the last replanning round
    vs the oracle's 10-step Euler (flowpolicy.py:273-292) on the fp32 model."""
    import numpy as np

    from oracle import pi0_oracle as po
    from oracle import pi0_torch as pt
    from oracle import specflow_oracle as so

    ids = [lo + int(i) for i in envs_local]
    ref = pt.Pi0Torch(po.AEConfig(), seed=0, kv_seed=1, env_ids=ids, device=dev)
    sel = list(envs_local)
    d_dev = draft[sel].double().cpu().numpy()
    import torch

    obs_s = torch.stack([torch.from_numpy(env_inputs(e)[0]) for e in ids]).to(dev)
    d_ref = ref.draft_forward(obs_s, gripper_bias=GRIP).double().cpu().numpy()
    draft_err = float(np.abs(d_dev - d_ref).max() / max(np.abs(d_ref[..., :-1]).max(), 1e-30))
    eps = eps_v[sel].double().cpu().numpy()
    st = state[sel]
    xs = np.stack([[so.interpolate(d_dev[i], eps[i], t) for t in TAUS] for i in range(len(sel))])
    xs = torch.from_numpy(xs.astype(np.float32)).to(dev)
    vm = ref.velocity(xs, TAUS, st, mirror_bf16=True).double().cpu().numpy()
    v32 = ref.velocity(xs, TAUS, st, mirror_bf16=False).double().cpu().numpy()
    rc, dc = recon[sel].double().cpu().numpy(), dist[sel].double().cpu().numpy()
    bc, res = branch[sel].cpu().numpy(), result[sel].cpu().numpy()
    sg = signs[sel].cpu().numpy()
    flips, near, margins, errs, refs, derr = 0, 0, [], [], [], 0.0
    for i in range(len(sel)):
        def ver(v):
            lut = {t: v[k] for k, t in enumerate(TAUS)}
            return so.verify(lambda x, t: lut[t], d_dev[i], eps[i], TAUS, vcfg.delta, 31, "l2", WINDOW,
                             float(sg[i]))
        rm, r32 = ver(vm[i]), ver(v32[i])
        path, planned = so.fallback_decision(rm["prefix"], rm["gripper_switch_detected"], 50,
                                             replan_size=REPLAN)
        code = ("flash_accepted", "flash_rejected_fallback", "flash_phase_fallback").index(path)
        rows = np.concatenate([rm["distances"][k, :min(rm["branch_prefixes"][k] + 1, 50)] for k in range(4)])
        m = float(np.abs(rows - vcfg.delta).min())
        near += m < 1e-4
        same = (tuple(int(x) for x in bc[i]) == rm["branch_prefixes"]
                and bool(res[i, 1]) == rm["gripper_switch_detected"] and int(res[i, 2]) == code
                and int(res[i, 3]) == planned)
        if not same:
            flips += 1
            margins.append(m)
        errs.append(rc[i] - r32["reconstructed"])
        refs.append(r32["reconstructed"])
        derr = max(derr, float(np.abs(dc[i] - rm["distances"]).max()))
    err, refa = np.stack(errs), np.stack(refs)
    rms = float(np.sqrt((refa ** 2).mean()))
    typ = np.abs(refa) >= rms
    euler = []
    if round_chunk is not None:
        paths = round_path.cpu().numpy()
        for j, i in enumerate(sel):
            if paths[i] == 0 or len(euler) == 2:
                continue
            e_idx = [j]
            st1 = state[i:i + 1]
            want = so.integrate_flow(
                lambda x, t: ref.velocity(torch.from_numpy(x.astype(np.float32))[None, None].to(dev), (t,), st1,
                                          mirror_bf16=False, env_index=e_idx)[0, 0].double().cpu().numpy(),
                eps_d[i].double().cpu().numpy(), 10)
            got = round_chunk[i].double().cpu().numpy()
            euler.append({"env": lo + int(i), "rel_norm_err_vs_fp32": float(np.linalg.norm(got - want) /
                                                                             np.linalg.norm(want))})
    return {"checked_envs": ids, "flips": flips, "flip_margins": margins, "near_threshold": int(near),
            "fallback_chunk_vs_fp32_euler": euler,
            "dist_max_abs_err_vs_bf16_oracle": derr,
            "recon_max_err_over_rms_vs_fp32": float(np.abs(err).max() / rms),
            "recon_max_rel_err_typical_vs_fp32": float((np.abs(err) / np.abs(refa))[typ].max()),
            "draft_max_err_rel": draft_err,
            "oracle": "oracle/pi0_torch.py (bf16-mirroring for decisions, unrounded fp32 for endpoints) + "
                      "oracle/specflow_oracle.py (reference verify / decision)"}


def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_13778_b200 import _capi
    from paper_2605_13778_b200.pi0 import PI0, ActionExpert, BatchedReplanner
    from paper_2605_13778_b200.sharding import gather_counts, max_over_ranks, shard_range
    from paper_2605_13778_b200.verifier import VerifierConfig

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    hbm_peak, tc_peak, tc_sust, peak_kind = peaks()
    cfg = PI0
    lo, hi = shard_range(args.envs, rank, world)
    E = hi - lo
    assert E >= 1, "more GPUs than environments"
    H, D, K = cfg.horizon, cfg.action_dim, len(TAUS)
    # weights replicated per GPU; each rank holds only its envs' prefix KV
    ae = ActionExpert(cfg, seed=0, n_envs=E, kv_seed=1, env_offset=lo, draft_gripper_bias=GRIP)
    obs_h, eps_v_h, eps_d_h, state_h, signs_h = shard_inputs(lo, hi)
    t = lambda a: torch.from_numpy(a).to(dev)
    obs, eps_v, eps_d, state, signs = map(t, (obs_h, eps_v_h, eps_d_h, state_h, signs_h))

    if args.calibrate:
        big = VerifierConfig(timesteps=TAUS, delta=1e30, gripper_window=WINDOW)
        _, _, dd, _, _ = ae.flash_batch(big, obs, eps_v, state, signs)
        m = dd[:, :, 0].amax(1)
        if world > 1:
            allm = [torch.empty_like(m) for _ in range(world)]
            dist.all_gather(allm, m)
            m = torch.cat(allm)
        if rank == 0:
            mm = m.cpu().numpy()[0::2]
            print(json.dumps({"calibrate": True, "quantiles": {str(q): float(np.quantile(mm, q))
                                                               for q in (0.25, 0.5, 0.75)}}))
        return

    vcfg = VerifierConfig(timesteps=TAUS, delta=DELTA_CFG4, gripper_window=WINDOW)
    outs = (torch.empty((E, H, D), device=dev), torch.empty((E, K, H, D), device=dev),
            torch.empty((E, K, H), device=dev), torch.empty((E, K), dtype=torch.int32, device=dev),
            torch.empty((E, 8), dtype=torch.int32, device=dev))

    def spec_step():
        ae.flash_batch(vcfg, obs, eps_v, state, signs, replan_size=REPLAN, outputs=outs)

    rp = BatchedReplanner(ae, E, vcfg, replan_size=REPLAN, periodic_refresh=PF)
    paths_acc = torch.zeros(5, dtype=torch.int64, device=dev)
    fb_rounds = torch.zeros(1, dtype=torch.int64, device=dev)
    fl_rounds = torch.zeros(2, dtype=torch.int64, device=dev)  # rounds with an attempt / with a compacted one
    fl_max_sub = []  # largest flash bucket below E (host value of the built graph)

    def round_step():
        _, path, _, _, _ = rp.round(obs, eps_v, eps_d, state, signs)
        if not fl_max_sub:
            fl_max_sub.append(rp.kernel_counts()[3])
        paths_acc.add_(torch.bincount(path.long(), minlength=5)[:5])
        fb_rounds.add_((rp.n_fallback > 0).long())
        n_att = (path <= 2).sum()
        fl_rounds[0].add_((n_att > 0).long())
        fl_rounds[1].add_(((n_att > 0) & (n_att <= fl_max_sub[0])).long())

    # ---------------- warm-up: round 0 is a full round for every env (no context
    # yet); later rounds settle into the flash / periodic / fallback mix
    for _ in range(max(3, args.warmup)):
        round_step()
        spec_step()
    torch.cuda.synchronize()
    paths_acc.zero_()
    fb_rounds.zero_()
    fl_rounds.zero_()

    # ---------------- timed region: replanning rounds (device time, max over ranks)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _capi.launch_count()
    with ClockSampler([local]) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            round_step()
        b.record()
        b.synchronize()
    # the flash-attempt and Euler bucket bodies of the graph SWITCHes run only
    # when selected: their kernels are added per round that ran them (device
    # counters); the host counter holds the fixed kernels + staging launches
    kc = rp.kernel_counts()
    fl = fl_rounds.tolist()
    launches = (_capi.launch_count() - launches0 + int(fb_rounds.item()) * kc[2] + fl[0] * kc[1] + fl[1] * 2)
    ms = max_over_ranks(a.elapsed_time(b) / args.steps, dev)
    path_counts = gather_counts(paths_acc.clone()).tolist()
    value = args.envs / (ms / 1e3)

    # ---------------- speculative attempt alone (the flash graph)
    if world > 1:
        dist.barrier()
    spec_ms = max_over_ranks(event_ms(spec_step, args.steps), dev)
    from paper_2605_13778_b200.sharding import decision_counts

    spec_counts = gather_counts(decision_counts(outs[4])).tolist()

    # ---------------- e2e through the public API with host buffers
    pin = lambda x: x.cpu().pin_memory()
    h_in = [pin(x) for x in (obs, eps_v, eps_d, state, signs)]
    d_in = [torch.empty_like(x) for x in (obs, eps_v, eps_d, state, signs)]
    h_chunk = torch.empty((E, H, D)).pin_memory()
    h_path = torch.empty(E, dtype=torch.int32).pin_memory()
    h_planned = torch.empty(E, dtype=torch.int32).pin_memory()

    def e2e_step():
        for h, d in zip(h_in, d_in):
            d.copy_(h, non_blocking=True)
        chunk, path, planned, _, _ = rp.round(*d_in)
        h_chunk.copy_(chunk, non_blocking=True)
        h_path.copy_(path, non_blocking=True)
        h_planned.copy_(planned, non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = max_over_ranks(event_ms(e2e_step, args.steps), dev)
    h2d = sum(x.numel() * x.element_size() for x in h_in)
    d2h = h_chunk.numel() * 4 + h_path.numel() * 4 + h_planned.numel() * 4

    # ---------------- dominant kernel: layer-0 gate/up GEMM (41 % of the flash FLOPs)
    rows_alg = E * K * cfg.seg_len
    gu_flops = 2.0 * rows_alg * (2 * cfg.mlp) * cfg.width
    ae.time_op(E, K, 2, 3)
    torch.cuda.synchronize()
    gu_ms = event_ms(lambda: ae.time_op(E, K, 2, 1), 20)
    gu_tflops = gu_flops / (gu_ms / 1e3) / 1e12
    traffic, in_step = None, None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            traffic = pj.get("gate_up_gemm_dram_bytes")
            in_step = pj.get("gate_up_gemm_in_step_ms")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": "gemm_pair_kernel<GEGLU> (layer gate/up, 2-SM CTA pairs)",
                "achieved": gu_tflops, "peak": tc_peak, "unit": "TFLOP/s", "frac": gu_tflops / tc_peak,
                "traffic": traffic, "traffic_source": "profiles/ncu_summary.json (ncu --set full capture)",
                "peak_kind": f"{peak_kind} burst bf16", "algorithmic_flops_per_launch": gu_flops,
                "ms_per_launch": gu_ms, "ms_per_launch_in_step_ncu": in_step,
                "frac_in_step_ncu": (gu_flops / (in_step / 1e3) / 1e12 / tc_peak) if in_step else None,
                "timing_note": "achieved/frac from back-to-back launches of the planned layer-0 op (CUDA events); "
                               "frac_in_step_ncu from the kernel's duration inside a replanning round under "
                               "ncu (profiles/ncu_summary.json r2, ~1.42 GHz)"}

    # algorithmic FLOPs: flash attempt for every env + 10-step Euler for each fallback env
    T = cfg.seg_len
    lay = cfg.width * (cfg.q_heads * cfg.head_dim + 2 * cfg.head_dim) + cfg.q_heads * cfg.head_dim * cfg.width \
        + 2 * cfg.mlp * cfg.width + cfg.mlp * cfg.width
    per_row = 2.0 * (cfg.layers * lay + cfg.width * D)
    attn_row = 4.0 * cfg.q_heads * cfg.head_dim * cfg.layers

    def fwd_flops(rows_keys):
        return sum(r * per_row + attn_row * k for r, k in rows_keys)

    flash_env = fwd_flops([(K * T, 0)]) + attn_row * K * ((cfg.prefix_len + 1) + H * (cfg.prefix_len + T)) \
        + 2.0 * (cfg.draft_in * cfg.draft_hidden + cfg.draft_hidden ** 2 + cfg.draft_hidden * H * D)
    euler_env = 10 * (fwd_flops([(T, 0)]) + attn_row * ((cfg.prefix_len + 1) + H * (cfg.prefix_len + T)))
    fb_per_round = sum(path_counts[1:]) / args.steps
    round_f = args.envs * flash_env + fb_per_round * euler_env
    round_tflops = round_f / (ms / 1e3) / 1e12
    spec_tflops = args.envs * flash_env / (spec_ms / 1e3) / 1e12
    roofline_step = {"bound": "tensor", "kernel": "whole replanning round (all kernels)",
                     "achieved": round_tflops, "peak": tc_sust, "unit": "TFLOP/s",
                     "frac": round_tflops / tc_sust, "peak_kind": f"{peak_kind} sustained bf16",
                     "algorithmic_flops_per_step": round_f, "flash_flops_per_env": flash_env,
                     "euler_flops_per_fallback_env": euler_env, "fallback_envs_per_round": fb_per_round,
                     "spec_attempt_frac": spec_tflops / tc_sust}

    names = ("flash_accepted", "flash_rejected_fallback", "flash_phase_fallback", "full", "periodic_refresh")
    line = {
        "metric": METRIC, "value": value, "unit": "rounds/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, KV, obs, noise)",
        "config": {"workload": "cfg4: pi0-scale Action Expert replanning round (flash attempt + device "
                               "bookkeeping + Euler full path on fallback envs), envs sharded",
                   "envs_total": args.envs, "envs_per_gpu": E, "K": K, "taus": list(TAUS),
                   "H": H, "D": D, "prefix_tokens": cfg.prefix_len, "layers": cfg.layers,
                   "width": cfg.width, "params": cfg.n_params(), "delta": DELTA_CFG4,
                   "replan_size": REPLAN, "periodic_refresh": PF, "euler_steps": 10,
                   "l2": "inputs larger than L2 (627 MB weights + 14.7 MB KV per env per step)",
                   "parallelism": f"envs sharded dp{world}, no hot-path collective",
                   "scaling_note": "fixed 512 envs split across ranks"},
        "value_spec": {"value": args.envs / (spec_ms / 1e3), "unit": "speculative attempts/s",
                       "ms_per_step": spec_ms},
        "decisions": {n: c for n, c in zip(names, path_counts)},
        "decision_mix": {"spec_attempt": {n: c for n, c in zip(names[:3], spec_counts)}},
        "roofline": roofline,
        "roofline_step": roofline_step,
        "e2e": {"value": args.envs / (e2e_ms / 1e3), "unit": "rounds/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "api": "BatchedReplanner.round"},
        "gpu_launches": int(launches),
        "device_mem_gb": round((lambda fr: (fr[1] - fr[0]) / 1e9)(torch.cuda.mem_get_info(dev)), 1),
        "clocks": clk.summary(),
    }
    # deciding-distance quantile of delta over the same-sign envs (sanity of DELTA_CFG4)
    m = outs[2][:, :, 0].amax(1)
    acc_frac = float((m[0::2] <= DELTA_CFG4).float().mean().item())
    line["decision_mix"]["delta_quantile"] = acc_frac

    # ---------------- parity audit (rank 0, after timing)
    if rank == 0 and not args.no_audit:
        spec_step()
        torch.cuda.synchronize()
        n = min(args.audit_envs, E)
        sample = sorted({int(round(i * (E - 1) / max(n - 1, 1))) for i in range(n)})
        try:
            line["parity"] = audit(ae, vcfg, lo, outs[0], outs[1], outs[2], outs[3], outs[4], eps_v, state,
                                   signs, sample, dev, rp.chunk, rp.path, eps_d)
        except Exception as exc:  # the audit must never hide the timing line
            line["parity"] = {"error": repr(exc)}

    # ---------------- batch-1 latency (cfg3) + HBM roofline, single GPU only
    if world == 1 and not args.no_latency:
        line.update(latency_b1(ae, vcfg, obs, eps_v, state, signs, hbm_peak, peak_kind, dev))
        line["latency_tiny"] = latency_tiny()
        # speculative attempt vs batch size: tensor utilisation at batch >= 64
        # (north star: >= 50 % of bf16 peak), same graph entry point
        sweep = []
        for b in (1, 8, 64, 128, 256):
            if b > E:
                break
            ob = ae.flash_batch(vcfg, obs[:b], eps_v[:b], state[:b], signs[:b])
            for _ in range(3):
                ae.flash_batch(vcfg, obs[:b], eps_v[:b], state[:b], signs[:b], outputs=ob)
            t = p50_ms(lambda: ae.flash_batch(vcfg, obs[:b], eps_v[:b], state[:b], signs[:b], outputs=ob),
                       20 if b >= 64 else 50)
            tf = b * flash_env / (t / 1e3) / 1e12
            sweep.append({"envs": b, "ms": t, "attempts_per_s": b / (t / 1e3), "tflops": tf,
                          "frac_of_sustained_bf16": tf / tc_sust})
        line["flash_batch_sweep"] = sweep

    # ---------------- CPU baseline (rank 0, N=1 only, bounded sample)
    if world == 1 and not args.no_cpu_baseline and rank == 0:
        tot, paths = 0.0, []
        for e in range(args.cpu_sample_envs):
            p, dt = cpu_replan_round(e)
            tot += dt
            paths.append(p)
        line["cpu_baseline"] = {"value": args.cpu_sample_envs / tot, "unit": "rounds/s",
                                "cores": os.cpu_count() or 1, "kind": "port",
                                "sample": f"{args.cpu_sample_envs} env replanning rounds of the cfg4 workload "
                                          f"(envs 0..{args.cpu_sample_envs - 1}: {paths}), numpy oracle on "
                                          f"the host"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def latency_b1(ae, vcfg, obs, eps_v, state, signs, hbm_peak, peak_kind, dev):
    """cfg3 batch 1: device-resident p50s, plus the reference-facing plugin calls
    (verifier.verify / flowpolicy.integrate_flow on the ActionExpert field,
    numpy in / numpy out, verifier.py:109-150 / flowpolicy.py:273-292)."""
    import numpy as np
    import torch

    from paper_2605_13778_b200.actions import STANDARDIZED, ActionChunk
    from paper_2605_13778_b200.flowpolicy import ConditioningCache, DenoiseConfig, integrate_flow
    from paper_2605_13778_b200.verifier import verify

    cfg = ae.cfg
    H, D = cfg.horizon, cfg.action_dim
    o1 = ae.flash_batch(vcfg, obs[:1], eps_v[:1], state[:1], signs[:1])
    v1 = ae.verify_batch(vcfg, o1[0], eps_v[:1], state[:1], signs[:1])
    start = eps_v[:1].clone()
    for _ in range(5):
        ae.flash_batch(vcfg, obs[:1], eps_v[:1], state[:1], signs[:1], outputs=o1)
        ae.verify_batch(vcfg, o1[0], eps_v[:1], state[:1], signs[:1], outputs=v1)
        ae.denoise_batch(start, state[:1], 10)
    torch.cuda.synchronize()
    spec = p50_ms(lambda: ae.flash_batch(vcfg, obs[:1], eps_v[:1], state[:1], signs[:1], outputs=o1), 50)
    ver = p50_ms(lambda: ae.verify_batch(vcfg, o1[0], eps_v[:1], state[:1], signs[:1], outputs=v1), 50)
    full = p50_ms(lambda: ae.denoise_batch(start, state[:1], 10), 20)
    # plugin calls: numpy in, numpy out, host sync included (wall clock)
    draft = ActionChunk(values=o1[0][0].double().cpu().numpy(), layout=ae.layout, space=STANDARDIZED)
    cache = ConditioningCache(embedding=np.zeros(0), kv=0)
    st = state[0].double().cpu().numpy()
    rng = np.random.default_rng(0)
    for _ in range(3):
        verify(ae, draft, cache, st, vcfg, rng)
        integrate_flow(ae, cache, st, DenoiseConfig(10), rng)
    plug_v = host_p50_ms(lambda: verify(ae, draft, cache, st, vcfg, rng), 30)
    plug_f = host_p50_ms(lambda: integrate_flow(ae, cache, st, DenoiseConfig(10), rng), 10)
    bytes_ver = cfg.weight_bytes_streamed() + cfg.kv_bytes()
    gbs = bytes_ver / (ver / 1e3) / 1e9
    traffic = None  # DRAM bytes of one speculative round, summed over its kernels (ncu launch list)
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("verify_b1", {}).get("dram_bytes")
        except Exception:
            traffic = None
    return {
        "latency_b1": {"spec_round_p50_ms": spec, "verify_p50_ms": ver, "full_round_p50_ms": full,
                       "plugin_verify_p50_ms": plug_v, "plugin_integrate_flow_p50_ms": plug_f,
                       "config": "cfg3: batch 1, K=4, H=50, D=32, P=800, 10-step Euler; plugin = "
                                 "verifier.verify / flowpolicy.integrate_flow with numpy in/out"},
        "roofline_b1": {"bound": "hbm", "kernel": "whole verify graph (batch 1)", "achieved": gbs,
                        "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak, "traffic": traffic,
                        "traffic_source": "profiles/ncu_summary.json verify_b1 (spec round incl. draft; "
                                          "ncu launch list, cold caches per kernel)",
                        "algorithmic_bytes": bytes_ver, "peak_kind": f"{peak_kind} hbm copy"},
    }


def latency_tiny():
    """cfg1 (tiny dVLA: D=7, H=50, K=3) p50 through the reference-shaped API
    (runtime.flash_attempt / runtime.full_round, numpy in/out) next to the
    reference algorithm on the host (oracle port of propose + verify and
    encode_context + integrate_flow, numpy float64, 1 thread)."""
    import numpy as np

    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import precision
    from paper_2605_13778_b200.actions import ChannelLayout, Standardizer
    from paper_2605_13778_b200.draft import DraftModel
    from paper_2605_13778_b200.flowpolicy import ContextEncoder, ObsNormalizer, Observation, VelocityField
    from paper_2605_13778_b200.nets import init_mlp
    from paper_2605_13778_b200.runtime import (Models, RunnerState, RuntimePolicy, flash_attempt,
                                               full_round)
    from paper_2605_13778_b200.verifier import VerifierConfig

    h, lay = 50, ChannelLayout(3, 3)
    d = lay.dim
    rng = np.random.default_rng(0)
    enc_net = init_mlp([7, 64, 32], rng)
    field_net = init_mlp([h * d + 1 + 39 + 3, 256, 256, h * d], rng)
    draft_net = init_mlp([10, 160, 160, h * d], rng)
    norm = ObsNormalizer.identity(5, 3)
    enc = ContextEncoder(net=enc_net, n_tasks=2, normalizer=norm)
    field = VelocityField(net=field_net, horizon=h, dim=d, emb_dim=39, state_dim=3, layout=lay)
    draft = DraftModel(net=draft_net, layout=lay, horizon=h, n_tasks=2, normalizer=norm)
    models = Models(encoder=enc, field=field, standardizer=Standardizer(np.zeros(d), np.ones(d)), draft=draft)
    policy = RuntimePolicy(verifier_cfg=VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=1.42,
                                                       gripper_window=24))
    obs = Observation(world_features=rng.normal(size=5), task_id=1, robot_state=rng.normal(size=3))
    out = {"config": "cfg1: D=7 (3/3/1), H=50, K=3, field [393,256,256,350], draft [10,160,160,350], "
                     "numpy in/out through runtime.flash_attempt / runtime.full_round"}
    for prec in ("fp32", "fp64"):
        with precision(prec):
            _, cache, _ = full_round(obs, models, policy, 0, 0, 7)
            state = RunnerState(cache=cache)
            for _ in range(20):
                flash_attempt(obs, models, policy, state, 1, 7)
                full_round(obs, models, policy, 0, 0, 7)
            out[f"spec_round_p50_ms_{prec}"] = host_p50_ms(
                lambda: flash_attempt(obs, models, policy, state, 1, 7), 300)
            out[f"full_round_p50_ms_{prec}"] = host_p50_ms(lambda: full_round(obs, models, policy, 0, 0, 7), 300)
    out.update(tiny_kernel_p50(field_net, draft_net, enc_net, h, d, lay.continuous_dims))
    # the reference algorithm on the host (numpy float64)
    fw = [np.asarray(w) for w in field_net.weights]
    fb = [np.asarray(b) for b in field_net.biases]
    dws = [np.asarray(w) for w in draft_net.weights]
    dbs = [np.asarray(b) for b in draft_net.biases]
    ews = [np.asarray(w) for w in enc_net.weights]
    ebs = [np.asarray(b) for b in enc_net.biases]
    feats_d = draft.features(obs)
    feats_e = enc.features(obs)
    emb = so.encode_context(ews, ebs, feats_e)
    st = norm.norm_state(obs.robot_state)
    cfgv = policy.verifier_cfg

    def ref_spec():
        dv = so.propose(dws, dbs, feats_d, h, d)
        e = np.random.default_rng(1).standard_normal((h, d))
        so.verify(lambda x, t: so.mlp_field_velocity(fw, fb, x, t, emb, st), dv, e, cfgv.timesteps,
                  cfgv.delta, lay.continuous_dims, "l2", 24, -1.0)

    def ref_full():
        em = so.encode_context(ews, ebs, feats_e)
        a0 = np.random.default_rng(2).standard_normal((h, d))
        so.integrate_flow(lambda x, t: so.mlp_field_velocity(fw, fb, x, t, em, st), a0, 10)

    out["cpu_reference_spec_round_p50_ms"] = host_p50_ms(ref_spec, 100)
    out["cpu_reference_full_round_p50_ms"] = host_p50_ms(ref_full, 100)
    out["cpu_reference_cores"] = 1
    out["cpu_reference_kind"] = "port (oracle/specflow_oracle.py, numpy float64)"
    out["cfg2"] = latency_cfg2()
    return out


def tiny_kernel_p50(field_net, draft_net, enc_net, h, d, cdims):
    """Device time of ONE fused launch (sf_tiny_flash_round: draft + K-branch
    verify + gate + decision; sf_tiny_full_round: encode + 10 Euler steps) on
    device-resident inputs, CUDA events around each launch, p50 of 200."""
    import torch

    from paper_2605_13778_b200 import _capi, _device, precision
    from paper_2605_13778_b200.verifier import VerifierConfig, make_cfg

    lib = _capi.lib()
    res = {}
    for prec in ("fp32", "fp64"):
        with precision(prec):
            dt = _device.tdtype()
            dev = torch.device("cuda")
            g = torch.Generator(device="cuda").manual_seed(0)
            feats, emb, state = (torch.randn(n, generator=g, device=dev).to(dt) for n in (10, 39, 3))
            eps = torch.randn(h * d, generator=g, device=dev).to(dt)
            outv = torch.empty(h * d * 5, dtype=dt, device=dev)
            words = torch.empty(32, dtype=torch.int32, device=dev)
            cfg = make_cfg(VerifierConfig(timesteps=(0.25, 0.5, 0.75), delta=1.42, gripper_window=24), -1.0)
            es = outv.element_size()
            o = _capi.SfVerifyOut(outv.data_ptr(), outv.data_ptr() + h * d * es, outv.data_ptr() + 4 * h * d * es,
                                  words.data_ptr() + 32, words.data_ptr())
            s_ = torch.cuda.current_stream().cuda_stream
            dd, fd, ed = draft_net.device().desc, field_net.device().desc, enc_net.device().desc

            def spec():
                _capi.check(lib.sf_tiny_flash_round(_device.code(), dd, feats.data_ptr(), fd, emb.data_ptr(), 39,
                                                    state.data_ptr(), 3, eps.data_ptr(), h, d, cdims, cfg, o, s_))

            def full():
                _capi.check(lib.sf_tiny_full_round(_device.code(), ed, feats.data_ptr(), 39, fd, state.data_ptr(), 3,
                                                   eps.data_ptr(), h, d, 10, outv.data_ptr(), None, words.data_ptr(),
                                                   s_))

            for fn in (spec, full):
                for _ in range(20):
                    fn()
            torch.cuda.synchronize()
            res[f"spec_round_kernel_p50_ms_{prec}"] = p50_ms(spec, 200)
            res[f"full_round_kernel_p50_ms_{prec}"] = p50_ms(full, 200)
    return res


def latency_cfg2():
    """cfg2: the reference-trained default policy (tests/golden/cfg2_*.ckpt,
    D=3, H=50, K=2, delta=0.15, N=10) on a recorded flash observation:
    runtime.flash_attempt / full_round p50 (numpy in/out, fp64) next to the
    reference algorithm's CPU p50 (oracle port, numpy float64, 1 thread)."""
    import numpy as np

    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import checkpoint as ck
    from paper_2605_13778_b200 import precision
    from paper_2605_13778_b200.draft import DraftModel
    from paper_2605_13778_b200.flowpolicy import ConditioningCache, ContextEncoder, ObsNormalizer, Observation
    from paper_2605_13778_b200.runtime import Models, RunnerState, RuntimePolicy, flash_attempt, full_round
    from paper_2605_13778_b200.verifier import VerifierConfig

    gold = ROOT / "tests" / "golden"
    tr = np.load(gold / "cfg2_trace.npz")
    enc, field, std, _ = ck.load_main_checkpoint(gold / "cfg2_main.ckpt")
    draft, _ = ck.load_draft_checkpoint(gold / "cfg2_draft.ckpt")
    ident = ObsNormalizer.identity(5, 3)
    models = Models(encoder=ContextEncoder(net=enc.net, n_tasks=enc.n_tasks, normalizer=ident), field=field,
                    standardizer=std, draft=DraftModel(net=draft.net, layout=draft.layout, horizon=draft.horizon,
                                                       n_tasks=draft.n_tasks, normalizer=ident))
    cfg = VerifierConfig(timesteps=tuple(tr["taus"]), delta=float(tr["delta"]), gripper_window=int(tr["window"]))
    policy = RuntimePolicy(verifier_cfg=cfg)
    i = int(np.nonzero(tr["call_kind"] == 1)[0][0])
    f = tr["call_dfeat"][i]
    obs = Observation(world_features=f[:5], task_id=int(np.argmax(f[5:7])), robot_state=f[7:10])
    st = RunnerState(cache=ConditioningCache(tr["call_emb"][i]), gripper_sign=float(tr["call_sign"][i]))
    out = {"config": "cfg2: reference-trained D=3, H=50, K=2 policy, recorded observation, fp64"}
    with precision("fp64"):
        for _ in range(20):
            flash_attempt(obs, models, policy, st, 1, 7)
            full_round(obs, models, policy, 0, 0, 7)
        out["spec_round_p50_ms"] = host_p50_ms(lambda: flash_attempt(obs, models, policy, st, 1, 7), 300)
        out["full_round_p50_ms"] = host_p50_ms(lambda: full_round(obs, models, policy, 0, 0, 7), 300)
    fw, fb = [np.asarray(w) for w in field.net.weights], [np.asarray(b) for b in field.net.biases]
    dws, dbs = [np.asarray(w) for w in draft.net.weights], [np.asarray(b) for b in draft.net.biases]
    ews, ebs = [np.asarray(w) for w in enc.net.weights], [np.asarray(b) for b in enc.net.biases]
    emb, state, sign = tr["call_emb"][i], f[7:10], float(tr["call_sign"][i])

    def ref_spec():
        dv = so.propose(dws, dbs, f, 50, 3)
        e = np.random.default_rng(1).standard_normal((50, 3))
        so.verify(lambda x, t: so.mlp_field_velocity(fw, fb, x, t, emb, state), dv, e, cfg.timesteps, cfg.delta,
                  2, "l2", cfg.gripper_window, sign)

    def ref_full():
        em = so.encode_context(ews, ebs, f[:7])
        a0 = np.random.default_rng(2).standard_normal((50, 3))
        so.integrate_flow(lambda x, t: so.mlp_field_velocity(fw, fb, x, t, em, state), a0, 10)

    out["cpu_reference_spec_round_p50_ms"] = host_p50_ms(ref_spec, 100)
    out["cpu_reference_full_round_p50_ms"] = host_p50_ms(ref_full, 100)
    out["cpu_reference_cores"] = 1
    return out


# --------------------------------------------------------------- cfg5 sweep

CFG5_DELTAS = (0.0, 0.05, 0.1, 0.15, 0.2, 0.3)   # PAPER.md:684-691 grid
CFG5_KS = (1, 2, 4, 8)
CFG5_HS = (16, 50, 100)


def sweep_tiny():
    """cfg5 on the tiny trained policy: the reference's own models re-trained
    per chunk horizon (tests/golden/cfg5_h{16,100}_*.ckpt, cfg2_*.ckpt for H =
    50; specflow.bench.cli run --seed 7 with chunk.horizon = H), replayed on the
    330 recorded flash-attempt observations of the reference's cfg2 episodes
    (draft / encoder features, normalised state, current gripper sign; the
    noise is re-drawn per H from the recorded verify seeds, verifier.py:129).
    Per (H, K): device p50 of one fused flash attempt (runtime.flash_attempt's
    device path, numpy in / out) next to the reference algorithm's CPU p50 (oracle
    port, numpy float64, 1 thread); per (H, K, delta): mean accepted prefix and
    accept / rejected / phase-fallback rates (runtime.py:286-320)."""
    import numpy as np

    from oracle import specflow_oracle as so
    from paper_2605_13778_b200 import checkpoint as ck
    from paper_2605_13778_b200 import precision
    from paper_2605_13778_b200.flowpolicy import ConditioningCache, _run_full
    from paper_2605_13778_b200.verifier import VerifierConfig, tiny_flash_round

    gold = ROOT / "tests" / "golden"
    tr = np.load(gold / "cfg2_trace.npz")
    sel = np.nonzero(tr["call_kind"] == 1)[0]
    rows = []
    for H in CFG5_HS:
        main = gold / ("cfg2_main.ckpt" if H == 50 else f"cfg5_h{H}_main.ckpt")
        dr = gold / ("cfg2_draft.ckpt" if H == 50 else f"cfg5_h{H}_draft.ckpt")
        enc, field, std, _ = ck.load_main_checkpoint(main)
        draft, _ = ck.load_draft_checkpoint(dr)
        lay = field.layout
        D = lay.dim
        with precision("fp64"):
            embs = [(_run_full(enc.net, tr["call_efeat"][i], enc.embed_dim, None, np.zeros(0), np.zeros(1), 1, 1,
                               0)[1]) for i in sel]
            for K in CFG5_KS:
                taus = tuple((k + 1) / (K + 1) for k in range(K))
                stats = []
                for delta in CFG5_DELTAS:
                    cfg = VerifierConfig(timesteps=taus, delta=delta, gripper_window=24)
                    L, paths = [], []
                    for j, i in enumerate(sel):
                        eps = np.random.default_rng(int(tr["call_seed"][i])).standard_normal((H, D))
                        _, rep = tiny_flash_round(field, draft.net, tr["call_dfeat"][i], ConditioningCache(embs[j]),
                                                  tr["call_state"][i], eps, cfg, float(tr["call_sign"][i]), lay)
                        L.append(rep.prefix)
                        paths.append(rep.decision)
                    n = len(paths)
                    stats.append({"delta": delta, "mean_prefix": float(np.mean(L)),
                                  "accept_rate": paths.count("flash_accepted") / n,
                                  "rejected_rate": paths.count("flash_rejected_fallback") / n,
                                  "phase_fallback_rate": paths.count("flash_phase_fallback") / n})
                i0 = int(sel[0])
                eps0 = np.random.default_rng(int(tr["call_seed"][i0])).standard_normal((H, D))
                cfg = VerifierConfig(timesteps=taus, delta=0.15, gripper_window=24)
                dev_ms = host_p50_ms(lambda: tiny_flash_round(
                    field, draft.net, tr["call_dfeat"][i0], ConditioningCache(embs[0]), tr["call_state"][i0], eps0,
                    cfg, float(tr["call_sign"][i0]), lay), 200)
                fw = [np.asarray(w) for w in field.net.weights]
                fb = [np.asarray(b) for b in field.net.biases]
                dws = [np.asarray(w) for w in draft.net.weights]
                dbs = [np.asarray(b) for b in draft.net.biases]

                def ref():
                    dv = so.propose(dws, dbs, tr["call_dfeat"][i0], H, D)
                    so.verify(lambda x, t: so.mlp_field_velocity(fw, fb, x, t, embs[0], tr["call_state"][i0]),
                              dv, eps0, taus, 0.15, lay.continuous_dims, "l2", 24, float(tr["call_sign"][i0]))

                cpu_ms = host_p50_ms(ref, 100)
                rows.append({"H": H, "K": K, "taus": list(taus), "spec_round_p50_ms_device_fp64": dev_ms,
                             "spec_round_p50_ms_cpu_reference": cpu_ms, "attempts": int(len(sel)),
                             "delta_sweep": stats})
    return {"workload": "cfg5 tiny: reference-trained D=3 models per H, 330 recorded flash observations",
            "cpu_reference": "oracle/specflow_oracle.py (numpy float64), 1 thread", "rows": rows}


def sweep_pi0(envs=64):
    """cfg5 at pi0 scale (random-init AE, bf16): batch-1 spec round / verify p50
    per (H, K), and over `envs` envs the accepted prefix / fallback rates at
    delta quantiles of the observed distances (random drafts with a one-signed
    gripper column so the phase gate does not mask the threshold sweep)."""
    import dataclasses

    import numpy as np
    import torch

    from paper_2605_13778_b200 import _capi
    from paper_2605_13778_b200.pi0 import PI0, ActionExpert
    from paper_2605_13778_b200.verifier import VerifierConfig

    rows = []
    for H in CFG5_HS:
        cfg = dataclasses.replace(PI0, horizon=H)
        ae = ActionExpert(cfg, n_envs=envs, draft_gripper_bias=GRIP)
        g = torch.Generator(device="cuda").manual_seed(H)
        D, S, F = cfg.action_dim, cfg.state_dim, cfg.draft_in
        obs = torch.randn((envs, F), generator=g, device="cuda")
        eps = torch.randn((envs, H, D), generator=g, device="cuda")
        state = torch.randn((envs, S), generator=g, device="cuda")
        signs = torch.ones(envs, device="cuda")
        for K in CFG5_KS:
            taus = tuple((k + 1) / (K + 1) for k in range(K))
            vc = VerifierConfig(timesteps=taus, delta=0.15, gripper_window=24)
            o1 = ae.flash_batch(vc, obs[:1], eps[:1], state[:1], signs[:1])
            for _ in range(3):
                ae.flash_batch(vc, obs[:1], eps[:1], state[:1], signs[:1], outputs=o1)
            torch.cuda.synchronize()
            spec = p50_ms(lambda: ae.flash_batch(vc, obs[:1], eps[:1], state[:1], signs[:1], outputs=o1), 20)
            draft, _, dist, _, _ = ae.flash_batch(vc, obs, eps, state, signs)
            d = dist.float().cpu().numpy()
            sweep = []
            for q in (0.0, 0.1, 0.25, 0.5, 0.75, 0.9):
                delta = float(np.quantile(d, q)) if q > 0 else 0.0
                _, _, _, res = ae.verify_batch(VerifierConfig(timesteps=taus, delta=delta, gripper_window=24),
                                               draft, eps, state, signs)
                r = res.cpu().numpy()
                path = r[:, _capi.SF_RES_PATH]
                sweep.append({"distance_quantile": q, "delta": delta,
                              "mean_prefix": float(r[:, _capi.SF_RES_PREFIX].mean()),
                              "accept_rate": float((path == _capi.SF_PATH_FLASH_ACCEPTED).mean()),
                              "rejected_rate": float((path == _capi.SF_PATH_FLASH_REJECTED).mean()),
                              "phase_fallback_rate": float((path == _capi.SF_PATH_FLASH_PHASE).mean())})
            rows.append({"H": H, "K": K, "taus": list(taus), "spec_round_b1_p50_ms": spec, "envs": envs,
                         "delta_sweep": sweep})
        del ae
        torch.cuda.empty_cache()
    return {"workload": "cfg5 pi0-scale (random-init AE, bf16, 1 GPU)", "rows": rows}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(respawn(args))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.sweep:
        if rank == 0:
            print(json.dumps({"metric": "cfg5 sweep: latency vs K, H; accepted prefix / fallback rate vs delta",
                              "tiny": sweep_tiny(), "pi0": sweep_pi0()}), flush=True)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
