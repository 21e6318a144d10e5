#!/bin/bash
# conflict-free staging: transforms k-core stride +16 B, pgrad row-group stride 144 B; bitwise vs
# lib_old, variants, A/B; ncu of the backward gather (retry) and of pgrad / transforms
export PYTHONPATH=$PWD
mkdir -p gpurun_out
P=$PWD/paper_2308_10087_b200
timeout 600 python tools/ab_bitwise.py $P/lib_old $P/lib --workload reddit > gpurun_out/j95_ab.txt 2>&1; echo "ab reddit rc=$?"; grep bitwise gpurun_out/j95_ab.txt
timeout 600 python tools/ab_bitwise.py $P/lib_old $P/lib --workload er >> gpurun_out/j95_ab.txt 2>&1; echo "ab er rc=$?"; grep bitwise gpurun_out/j95_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -m gpu -p no:cacheprovider -x > gpurun_out/j95_tests.txt 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/j95_tests.txt
for rep in 1 2; do
for K in 4 32; do
for L in lib lib_old; do
  GP_LIBDIR=$P/$L timeout 400 python bench.py --chunks $K --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j95_b_K${K}_${L}_r$rep.json 2> gpurun_out/j95_b_K${K}_${L}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j95_b_K${K}_${L}_r$rep.json')); k=d['kernel_ms_per_epoch']; print('K=$K $L rep=$rep', round(d['value'],4), 'pgrad', k['pgrad'], 'fwd_dense', k['fwd_dense'], 'bwd_dense', k['bwd_dense'])"
done; done; done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_bwd8" --launch-skip 40 -c 3 -f -o gpurun_out/j95_ncu_bwd python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/j95_ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"; tail -3 gpurun_out/j95_ncu_bwd.log
timeout 600 ncu --set full --clock-control none -k "regex:k_tc_xform|k_pgrad_tc" --launch-skip 40 -c 4 -f -o gpurun_out/j95_ncu_tc python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu tc rc=$?"
timeout 600 ncu --set full --clock-control none -k "regex:k_pgrad_tc" --launch-skip 10 -c 2 -f -o gpurun_out/j95_ncu_pgrad python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu pgrad rc=$?"
for r in bwd tc pgrad; do
  ncu -i gpurun_out/j95_ncu_$r.ncu-rep --page details --csv > gpurun_out/j95_ncu_${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/j95_ncu_$r.ncu-rep --page raw --csv > gpurun_out/j95_ncu_${r}_raw.csv 2>/dev/null
  rm -f gpurun_out/j95_ncu_$r.ncu-rep
done
