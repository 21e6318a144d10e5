#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/e2e_probe.py 2>&1 | tail -3
GP_SPLIT=0 timeout 600 python tools/e2e_probe.py 2>&1 | tail -3
for k in "k_fwd8<.int.2, .int.2, .bool.1>" "k_fwd_tile<.bool.1, .int.4>" "k_bwd8<.int.1, .int.0, .int.2, .bool.1>" "k_bwd_tile<.int.4>"; do
  n=$(echo "$k" | tr -cd 'a-z0-9_')
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$k" -s 40 -c 1 -o gpurun_out/j21_$n python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/j21_ncu_$n.log 2>&1; echo "$k rc=$?"; grep -c "No kernels" gpurun_out/j21_ncu_$n.log
done
