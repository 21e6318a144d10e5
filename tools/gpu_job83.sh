#!/bin/bash
# racecheck over the parity tests job 82 did not reach (hybrid, powerlaw, ledger, determinism, ...)
export PYTHONPATH=$PWD
timeout 1700 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest $(cat tools/racecheck_rest.txt) -q -m gpu -p no:cacheprovider > gpurun_out/j83_racecheck.txt 2>&1; echo "racecheck rc=$?"; grep -E "passed|failed|SUMMARY|skipped" gpurun_out/j83_racecheck.txt | tail -3
