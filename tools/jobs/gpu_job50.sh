#!/bin/bash
export PYTHONPATH=$PWD
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pgrad_tc -s 20 -c 1 -o gpurun_out/j50_pgrad python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/j50.log 2>&1; echo rc=$?
