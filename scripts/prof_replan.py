"""ncu launch list of one cfg4 replanning round. ncu cannot profile the kernel
nodes of a graph that holds conditional nodes (the round's Euler SWITCH), so
after warm-up rounds the same work is replayed as its two plain graphs between
cudaProfilerStart/Stop: the flash attempt on the flash bucket the round
selected (sf_ae_flash_round on that many envs: the attempting envs are
compacted into it) and the 10-step Euler on the Euler bucket the round
selected (sf_ae_denoise_envs on the compacted fallback envs) -- the kernels
the two SWITCH bodies run.

usage: ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
         --log-file gpurun_out/replan_launches.csv python scripts/prof_replan.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

import bench
from paper_2605_13778_b200.pi0 import PI0, ActionExpert, BatchedReplanner
from paper_2605_13778_b200.verifier import VerifierConfig


def main():
    E = 512
    ae = ActionExpert(PI0, n_envs=E, kv_seed=1, draft_gripper_bias=bench.GRIP)
    obs, ev, ed, st, sg = (torch.from_numpy(x).cuda() for x in bench.shard_inputs(0, E))
    vc = VerifierConfig(timesteps=bench.TAUS, delta=bench.DELTA_CFG4, gripper_window=bench.WINDOW)
    rp = BatchedReplanner(ae, E, vc, replan_size=bench.REPLAN, periodic_refresh=bench.PF)
    for _ in range(4):
        rp.round(obs, ev, ed, st, sg)
    torch.cuda.synchronize()
    n_fb = int(rp.n_fallback.item())
    n_att = int((rp.path <= 2).sum().item())
    fbucket = min(b for b in ([1, 2, 4, 8, 16] + list(range(32, E, 32)) + [E]) if b >= max(n_att, 1))
    bucket = min(b for b in ([1, 2, 4, 8, 16, 32] + list(range(64, E + 64, 64))) if b >= n_fb)
    idx = torch.nonzero(rp.path != 0).flatten().to(torch.int32)
    idx = torch.cat([idx, idx[:1].repeat(bucket - len(idx))]).contiguous()
    start, state = ed[idx.long()].contiguous(), st[idx.long()].contiguous()
    for _ in range(2):
        ae.flash_batch(vc, obs[:fbucket], ev[:fbucket], st[:fbucket], sg[:fbucket], replan_size=bench.REPLAN)
        ae.denoise_envs(idx, start, state, 10)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    ae.flash_batch(vc, obs[:fbucket], ev[:fbucket], st[:fbucket], sg[:fbucket], replan_size=bench.REPLAN)
    ae.denoise_envs(idx, start, state, 10)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("attempting envs:", n_att, "flash bucket:", fbucket, "fallback envs:", n_fb, "bucket:", bucket)


if __name__ == "__main__":
    main()
