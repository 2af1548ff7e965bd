#!/bin/bash
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_b1engine_gpu.py"
for tool in memcheck synccheck racecheck; do
  out=gpurun_out/sanitizer_engine_${tool}.log
  echo "== $tool (batch-1 engine)" > $out
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest $SEL -q -x -p no:cacheprovider -k "not 10" >> $out 2>&1
  echo "rc=$?" >> $out
done
