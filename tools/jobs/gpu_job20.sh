#!/bin/bash
# Evidence for the split default: bench line, launch list, ncu --set full of the four row kernels.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/j20_bench.json 2> gpurun_out/j20_bench.err; tail -c 400 gpurun_out/j20_bench.json
timeout 600 python bench.py --steps 5 --warmup 3 --chunks 32 --no-e2e --no-cpu-baseline > gpurun_out/j20_K32.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j20_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launch list rc=$?"
for k in "k_fwd8<2, 2, 1>" "k_fwd_tile<1, 4>" "k_bwd8<1, 0, 2, 1>" "k_bwd_tile<4>"; do
  n=$(echo "$k" | tr -cd 'a-z0-9_')
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$k" -s 40 -c 1 -o gpurun_out/j20_$n python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/j20_ncu_$n.log 2>&1; echo "$k rc=$?"
done
