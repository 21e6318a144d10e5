#!/bin/bash
# compute-sanitizer over the smoke run (GCNII-5 epoch + 2-stage pipeline): memcheck, racecheck, synccheck
export PYTHONPATH=$PWD
for t in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j81_$t.txt 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/j81_$t.txt
done
