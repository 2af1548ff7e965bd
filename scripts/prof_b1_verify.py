"""ncu launch list of one batch-1 speculative round (cfg3: draft + K=4 verify
of the pi0-scale Action Expert, the flash_batch graph at n_envs = 1) between
cudaProfilerStart/Stop, for the DRAM traffic of the whole verify (bench.py
roofline_b1.traffic: dram__bytes_read + write summed over its kernels).

usage: ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
         --clock-control none --csv --log-file gpurun_out/b1_verify_launches.csv python scripts/prof_b1_verify.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

from paper_2605_13778_b200 import pi0
from paper_2605_13778_b200.verifier import VerifierConfig


def main():
    rng = np.random.default_rng(5)
    cuda = lambda a: torch.from_numpy(a.astype(np.float32)).cuda()  # noqa: E731
    obs, eps = cuda(rng.standard_normal((1, 64))), cuda(rng.standard_normal((1, 50, 32)))
    state, signs = cuda(rng.standard_normal((1, 32))), torch.ones(1, device="cuda")
    ae = pi0.ActionExpert(pi0.PI0, seed=0, n_envs=1, kv_seed=1)
    vc = VerifierConfig(timesteps=(0.2, 0.4, 0.6, 0.8), delta=5.64, gripper_window=24)
    out = ae.flash_batch(vc, obs, eps, state, signs)
    for _ in range(3):
        ae.flash_batch(vc, obs, eps, state, signs, outputs=out)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    ae.flash_batch(vc, obs, eps, state, signs, outputs=out)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
