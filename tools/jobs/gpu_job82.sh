#!/bin/bash
# compute-sanitizer over the GPU parity suite (every trainer, engine variant, layer kind): memcheck + racecheck
export PYTHONPATH=$PWD
for t in memcheck racecheck; do
timeout 1300 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider > gpurun_out/j82_$t.txt 2>&1; echo "$t rc=$?"; grep -E "passed|failed|SUMMARY" gpurun_out/j82_$t.txt | tail -3
done
