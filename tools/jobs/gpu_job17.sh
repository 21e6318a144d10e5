#!/bin/bash
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_fwd_tile -s 1 -c 1 -o gpurun_out/prof_tile4 ./tools/fwd_bench > gpurun_out/j17_ncu.log 2>&1; tail -1 gpurun_out/j17_ncu.log
ncu --set full --import-source on --clock-control none -k regex:k_fwd_tile -s 22 -c 1 -o gpurun_out/prof_tile4_k32 ./tools/fwd_bench > gpurun_out/j17b_ncu.log 2>&1; tail -1 gpurun_out/j17b_ncu.log
