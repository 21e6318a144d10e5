#!/bin/bash
# launch list of the final code (serialised ncu, per-kernel shares)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/j118_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/j118_ncu_list.log 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/j118_launches.csv "# ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 python bench.py --steps 1 --warmup 1 (session's final kernels)" > gpurun_out/j118_launches_summary.txt; head -24 gpurun_out/j118_launches_summary.txt
