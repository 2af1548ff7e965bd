"""Drive cfg4 replanning rounds for an ncu launch list: warm-up rounds, then
ONE round between cudaProfilerStart/Stop (run ncu with --profile-from-start off).

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
    torch.cuda.cudart().cudaProfilerStart()
    rp.round(obs, ev, ed, st, sg)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("fallback envs:", int(rp.n_fallback.item()))


if __name__ == "__main__":
    main()
