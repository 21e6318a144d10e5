#!/bin/bash
# transform staging with the padded k-core stride only (pgrad as before): bitwise vs lib_old, A/B x3
export PYTHONPATH=$PWD
mkdir -p gpurun_out
P=$PWD/paper_2308_10087_b200
timeout 600 python tools/ab_bitwise.py $P/lib_old $P/lib --workload er > gpurun_out/j91_ab.txt 2>&1; echo "ab er rc=$?"
timeout 600 python tools/ab_bitwise.py $P/lib_old $P/lib --workload reddit >> gpurun_out/j91_ab.txt 2>&1; echo "ab reddit rc=$?"; grep bitwise gpurun_out/j91_ab.txt
for rep in 1 2 3; do
for K in 32 4; do
for L in lib lib_old; do
  GP_LIBDIR=$P/$L timeout 400 python bench.py --chunks $K --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j91_b_K${K}_${L}_r$rep.json 2> gpurun_out/j91_b_K${K}_${L}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j91_b_K${K}_${L}_r$rep.json')); k=d['kernel_ms_per_epoch']; print('K=$K $L rep=$rep', round(d['value'],4), 'pgrad', k['pgrad'], 'fwd_dense', k['fwd_dense'], 'bwd_dense', k['bwd_dense'])"
done; done; done
