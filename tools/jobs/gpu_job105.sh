#!/bin/bash
# pgrad operand prefetch depth with conflict-free staging: PF 4 (lib) vs 2 vs 1 (the previous loop)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
P=$PWD/paper_2308_10087_b200
timeout 600 python tools/ab_bitwise.py $P/lib_pf1 $P/lib --workload reddit > gpurun_out/j105_ab.txt 2>&1; echo "ab rc=$?"; grep bitwise gpurun_out/j105_ab.txt
for rep in 1 2; do
for L in lib lib_pf2 lib_pf1; do
  GP_LIBDIR=$P/$L timeout 400 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j105_${L}_r$rep.json 2> gpurun_out/j105_${L}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j105_${L}_r$rep.json')); print('$L rep=$rep', round(d['value'],4), 'pgrad', d['kernel_ms_per_epoch']['pgrad'])"
done; done
