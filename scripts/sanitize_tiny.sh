#!/bin/bash
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_tiny_gpu.py::test_cfg1_flash_attempt_matches_reference tests/test_tiny_gpu.py::test_cfg1_verify_and_full_round tests/test_verifier_kats_gpu.py"
for tool in memcheck racecheck synccheck; do
  out=gpurun_out/sanitizer_tiny_${tool}.log
  echo "== $tool (tiny path, st.async all-gather)" > $out
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest $SEL -q -x -p no:cacheprovider >> $out 2>&1
  echo "rc=$?" >> $out
done
