#!/usr/bin/env python
"""Benchmark of the B200-native speculative-replanning path (driver contract).

Headline workload (BASELINE.json configs[3], "cfg4"): the pi0-scale Action
Expert (18 layers, width 1024, 8x256 MQA heads, GeGLU 4096; ~314M params,
bf16) over a per-env random-init VLM prefix KV cache (800 tokens), chunk
50 x 32, K = 4 verification timesteps; 512 synthetic environments sharded
across the GPUs (strong scaling, no collective on the hot path). One step =
one speculative round (draft MLP -> 4-branch verify -> longest-consistent
prefix -> gripper gate -> decision) for every env, replayed as one CUDA graph.

value      = speculative rounds / s over all GPUs (device time, max over ranks)
e2e        = the same through ActionExpert.flash_batch with HOST inputs:
             pinned H2D of obs/eps/state/signs + D2H of decisions every step
latency_b1 = cfg3 batch-1 p50 latencies (spec round, verify, 10-step full round)
roofline   = dominant kernel (gate/up GEMM, tensor-bound) + batch-1 verify (HBM)
cpu_baseline / --impl reference = the CPU oracle port of the reference path
             (oracle/: the reference's numpy algorithm driving the pi0 field)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "p50 speculative-round & full-round latency (ms); rounds/sec at 1/2/4/8 B200"
TAUS = (0.2, 0.4, 0.6, 0.8)
DELTA = 0.15
WINDOW = 24


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--envs", type=int, default=512, help="total environments (all GPUs)")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-envs", type=int, default=2)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


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


# --------------------------------------------------------------- CPU side

def cpu_rounds(n_envs: int, seed: int = 0):
    """The reference algorithm on the host: oracle/specflow_oracle.verify (the
    reference's Alg. 1, pinned to its goldens) driving the numpy pi0 field, one
    env after another (the reference is a sequential loop, harness.py:489-552).
    Returns (seconds, rounds)."""
    import numpy as np

    from oracle import pi0_oracle as po
    from oracle import specflow_oracle as so

    cfg = po.AEConfig()
    w = po.make_weights(cfg, 0)
    dw = po.make_draft_weights(cfg, 0)
    rng = np.random.default_rng(seed)
    kvs = [po.make_prefix_kv(cfg, 1, e) for e in range(n_envs)]
    t0 = time.perf_counter()
    for e in range(n_envs):
        obs = rng.standard_normal((1, cfg.draft_in)).astype(np.float32)
        eps = rng.standard_normal((cfg.horizon, cfg.action_dim))
        state = rng.standard_normal(cfg.state_dim).astype(np.float32)
        draft = po.draft_forward(cfg, dw, obs)[0].astype(np.float64)
        rep = so.verify(lambda x, t: po.field_velocity(cfg, w, kvs[e], [(x.astype(np.float32), t)],
                                                       state)[0],
                        draft, eps, TAUS, DELTA, cfg.action_dim - 1, "l2", WINDOW, -1.0)
        so.fallback_decision(rep["prefix"], rep["gripper_switch_detected"], cfg.horizon)
    return time.perf_counter() - t0, n_envs


def run_reference(args, rank, world):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    times = []
    for i in range(args.warmup + args.steps):
        dt, n = cpu_rounds(1, seed=i)
        if i >= args.warmup:
            times.append(dt / n)
    per = statistics.mean(times)
    value = 1.0 / per
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rounds/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "cfg4 speculative round per env (pi0-scale AE, K=4, H=50, D=32, P=800)",
                   "sample": "1 env round per step on the host CPU"},
        "cpu_baseline": {"value": value, "unit": "rounds/s", "cores": cores, "kind": "port",
                         "sample": "1 env speculative round per step (draft + 4-branch verify)"},
        "e2e": {"value": value, "unit": "rounds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU side

def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_13778_b200 import _capi
    from paper_2605_13778_b200.pi0 import PI0, ActionExpert
    from paper_2605_13778_b200.sharding import (decision_counts, gather_counts, max_over_ranks,
                                                shard_range)
    from paper_2605_13778_b200.verifier import VerifierConfig

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    hbm_peak, tc_peak, tc_sust, peak_kind = peaks()
    cfg = PI0
    lo, hi = shard_range(args.envs, rank, world)
    E = hi - lo
    assert E >= 1, "more GPUs than environments"
    # weights replicated per GPU; each rank holds only its envs' prefix KV
    ae = ActionExpert(cfg, seed=0, n_envs=E, kv_seed=1, env_offset=lo)
    vcfg = VerifierConfig(timesteps=TAUS, delta=DELTA, gripper_window=WINDOW)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    dev = torch.device("cuda", local)
    H, D, S, F = cfg.horizon, cfg.action_dim, cfg.state_dim, cfg.draft_in
    obs = torch.randn((E, F), generator=g, device=dev)
    eps = torch.randn((E, H, D), generator=g, device=dev)
    state = torch.randn((E, S), generator=g, device=dev)
    signs = torch.where(torch.rand(E, generator=g, device=dev) < 0.5, -1.0, 1.0)
    K = len(TAUS)
    outs = (torch.empty((E, H, D), device=dev), torch.empty((E, K, H, D), device=dev),
            torch.empty((E, K, H), device=dev), torch.empty((E, K), dtype=torch.int32, device=dev),
            torch.empty((E, 8), dtype=torch.int32, device=dev))

    def step():
        ae.flash_batch(vcfg, obs, eps, state, signs, outputs=outs)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region (device time, CUDA events, max over ranks)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _capi.launch_count()
    with ClockSampler([local]) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            step()
        b.record()
        b.synchronize()
    launches = _capi.launch_count() - launches0
    ms = max_over_ranks(a.elapsed_time(b) / args.steps, dev)
    # metrics gather after the timed region (the only data collective)
    counts = gather_counts(decision_counts(outs[4])).tolist()
    if world > 1:
        dist.barrier()
    value = args.envs / (ms / 1e3)

    # ---------------- e2e through the public API with host buffers
    h_obs, h_eps = obs.cpu().pin_memory(), eps.cpu().pin_memory()
    h_state, h_signs = state.cpu().pin_memory(), signs.cpu().pin_memory()
    d_obs, d_eps, d_state, d_signs = (torch.empty_like(x) for x in (obs, eps, state, signs))
    h_branch = torch.empty((E, K), dtype=torch.int32).pin_memory()
    h_res = torch.empty((E, 8), dtype=torch.int32).pin_memory()

    def e2e_step():
        d_obs.copy_(h_obs, non_blocking=True)
        d_eps.copy_(h_eps, non_blocking=True)
        d_state.copy_(h_state, non_blocking=True)
        d_signs.copy_(h_signs, non_blocking=True)
        o = ae.flash_batch(vcfg, d_obs, d_eps, d_state, d_signs, outputs=outs)
        h_branch.copy_(o[3], non_blocking=True)
        h_res.copy_(o[4], non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = max_over_ranks(event_ms(e2e_step, args.steps), dev)
    h2d = sum(x.numel() * x.element_size() for x in (h_obs, h_eps, h_state, h_signs))
    d2h = h_branch.numel() * 4 + h_res.numel() * 4

    # ---------------- dominant kernel: layer-0 gate/up GEMM (41% of the FLOPs)
    rows_alg = E * K * cfg.seg_len
    gu_flops = 2.0 * rows_alg * (2 * cfg.mlp) * cfg.width
    ae.time_op(E, K, 2, 3)
    torch.cuda.synchronize()
    gu_ms = event_ms(lambda: ae.time_op(E, K, 2, 1), 20)
    gu_tflops = gu_flops / (gu_ms / 1e3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("gate_up_gemm_dram_bytes")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": "gemm_pair_kernel<GEGLU> (layer gate/up, 2-SM CTA pairs)",
                "achieved": gu_tflops, "peak": tc_peak, "unit": "TFLOP/s", "frac": gu_tflops / tc_peak,
                "traffic": traffic, "peak_kind": f"{peak_kind} burst bf16",
                "algorithmic_flops_per_launch": gu_flops, "ms_per_launch": gu_ms}

    # whole-step tensor utilisation: algorithmic FLOPs of one speculative round
    # for every env (draft MLP + 18-layer verify over K branches + head) / step time
    T = cfg.seg_len
    lay = cfg.width * (cfg.q_heads * cfg.head_dim + 2 * cfg.head_dim) + cfg.q_heads * cfg.head_dim * cfg.width \
        + 2 * cfg.mlp * cfg.width + cfg.mlp * cfg.width
    gemm_f = 2.0 * rows_alg * (cfg.layers * lay + cfg.width * D)
    keys = K * ((cfg.prefix_len + 1) + H * (cfg.prefix_len + T))  # per env: state + action rows
    attn_f = 4.0 * E * keys * cfg.q_heads * cfg.head_dim * cfg.layers
    draft_f = 2.0 * E * (cfg.draft_in * cfg.draft_hidden + cfg.draft_hidden ** 2 + cfg.draft_hidden * H * D)
    step_f = gemm_f + attn_f + draft_f
    step_tflops = step_f / (ms / 1e3) / 1e12
    roofline_step = {"bound": "tensor", "kernel": "whole speculative-round step (all kernels)",
                     "achieved": step_tflops, "peak": tc_sust, "unit": "TFLOP/s",
                     "frac": step_tflops / tc_sust, "peak_kind": f"{peak_kind} sustained bf16",
                     "algorithmic_flops_per_step": step_f, "gemm_flops": gemm_f, "attn_flops": attn_f}

    line = {
        "metric": METRIC, "value": value, "unit": "rounds/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, KV, obs, noise)",
        "config": {"workload": "cfg4: pi0-scale Action Expert speculative round, envs sharded",
                   "envs_total": args.envs, "envs_per_gpu": E, "K": K, "taus": list(TAUS),
                   "H": H, "D": D, "prefix_tokens": cfg.prefix_len, "layers": cfg.layers,
                   "width": cfg.width, "params": cfg.n_params(), "delta": DELTA,
                   "l2": "inputs larger than L2 (627 MB weights + 14.7 MB KV per env per step)",
                   "parallelism": f"envs sharded dp{world}, no hot-path collective"},
        "roofline": roofline,
        "roofline_step": roofline_step,
        "decisions": {"flash_accepted": counts[0], "flash_rejected_fallback": counts[1],
                      "flash_phase_fallback": counts[2]},
        "e2e": {"value": args.envs / (e2e_ms / 1e3),
                "unit": "rounds/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": "ActionExpert.flash_batch"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }

    # ---------------- batch-1 latency (cfg3) + HBM roofline, single GPU only
    if world == 1 and not args.no_latency:
        o1 = ae.flash_batch(vcfg, obs[:1], eps[:1], state[:1], signs[:1])
        v1 = ae.verify_batch(vcfg, o1[0], eps[:1], state[:1], signs[:1])
        start = torch.randn((1, H, D), generator=g, device=dev)
        for _ in range(5):
            ae.flash_batch(vcfg, obs[:1], eps[:1], state[:1], signs[:1], outputs=o1)
            ae.verify_batch(vcfg, o1[0], eps[:1], state[:1], signs[:1], outputs=v1)
            ae.denoise_batch(start, state[:1], 10)
        torch.cuda.synchronize()
        spec = p50_ms(lambda: ae.flash_batch(vcfg, obs[:1], eps[:1], state[:1], signs[:1], outputs=o1), 50)
        ver = p50_ms(lambda: ae.verify_batch(vcfg, o1[0], eps[:1], state[:1], signs[:1], outputs=v1), 50)
        full = p50_ms(lambda: ae.denoise_batch(start, state[:1], 10), 20)
        bytes_ver = cfg.weight_bytes_streamed() + cfg.kv_bytes()
        gbs = bytes_ver / (ver / 1e3) / 1e9
        line["latency_b1"] = {"spec_round_p50_ms": spec, "verify_p50_ms": ver, "full_round_p50_ms": full,
                              "config": "cfg3: batch 1, K=4, H=50, D=32, P=800, 10-step Euler"}
        line["roofline_b1"] = {"bound": "hbm", "kernel": "whole verify graph (batch 1)",
                               "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                               "traffic": None, "algorithmic_bytes": bytes_ver,
                               "peak_kind": f"{peak_kind} hbm copy"}

    # ---------------- CPU baseline (rank 0, N=1 only, bounded sample)
    if world == 1 and not args.no_cpu_baseline and rank == 0:
        dt, n = cpu_rounds(args.cpu_sample_envs)
        line["cpu_baseline"] = {"value": n / dt, "unit": "rounds/s", "cores": os.cpu_count() or 1,
                                "kind": "port",
                                "sample": f"{n} env speculative rounds (draft + 4-branch verify) of "
                                          f"the cfg4 workload, numpy float32 on the host"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
