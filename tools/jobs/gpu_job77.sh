#!/bin/bash
# ncu --set full of the backward gathers (done-filtered AGG and unfiltered AGG_ALL), headline config
export PYTHONPATH=$PWD
for v in "1:agg" "6:agg_all"; do k=${v%%:*}; n=${v##*:}
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_bwd8<.int.$k, .int.0, .int.2, .bool.1, .int.5>" -s 20 -c 1 -o gpurun_out/j77_bwd_$n \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/j77_$n.log 2>&1; echo "ncu $n rc=$?"
done
ls -la gpurun_out/j77_*
