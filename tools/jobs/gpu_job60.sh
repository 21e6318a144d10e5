#!/bin/bash
# Final-state evidence: launch list and ncu --set full of the dominant kernel as the engine now runs it
# (5-CTA split gather for K=4 chunk launches).
export PYTHONPATH=$PWD
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j60_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_fwd8<.int.2, .int.2, .bool.1, .int.5>" -s 40 -c 1 -o gpurun_out/j60_fwd_occ5 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/j60_ncu.log 2>&1; echo "ncu rc=$?"; grep -c "No kernels" gpurun_out/j60_ncu.log
