#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the tiny path and the
# reduced pi0 chain. Logs -> gpurun_out/sanitizer_<tool>.log
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
SEL_TINY="tests/test_tiny_gpu.py::test_prefix_kernel_exhaustive_and_random tests/test_verifier_kats_gpu.py"
SEL_PI0="tests/test_pi0_gpu.py::test_velocity_matches_oracle_small tests/test_pi0_gpu.py::test_denoise_matches_oracle_small tests/test_pi0_gpu.py::test_replan_update_matches_run_episode_bookkeeping"
for tool in memcheck racecheck synccheck; do
  out=gpurun_out/sanitizer_${tool}.log
  echo "== $tool (tiny path)" > $out
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest $SEL_TINY -q -x -p no:cacheprovider >> $out 2>&1
  echo "rc=$?" >> $out
  echo "== $tool (pi0 chain, reduced shapes)" >> $out
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest $SEL_PI0 -q -x -p no:cacheprovider >> $out 2>&1
  echo "rc=$?" >> $out
done
