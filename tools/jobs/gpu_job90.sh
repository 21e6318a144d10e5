#!/bin/bash
# padded k-core strides in the tcgen05 staging buffers (pgrad, transforms): bitwise vs the
# previous build (lib_old), parity suites, A/B epoch time
export PYTHONPATH=$PWD
mkdir -p gpurun_out
P=$PWD/paper_2308_10087_b200
timeout 600 python tools/ab_bitwise.py $P/lib_old $P/lib --workload er > gpurun_out/j90_ab.txt 2>&1; echo "ab er rc=$?"
timeout 600 python tools/ab_bitwise.py $P/lib_old $P/lib --workload reddit >> gpurun_out/j90_ab.txt 2>&1; echo "ab reddit rc=$?"; cat gpurun_out/j90_ab.txt | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -m gpu -p no:cacheprovider > gpurun_out/j90_tests.txt 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/j90_tests.txt
for rep in 1 2; do
for K in 4 32; do
for L in lib lib_old; do
  GP_LIBDIR=$P/$L timeout 400 python bench.py --chunks $K --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j90_b_K${K}_${L}_r$rep.json 2> gpurun_out/j90_b_K${K}_${L}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j90_b_K${K}_${L}_r$rep.json')); k=d['kernel_ms_per_epoch']; print('K=$K $L rep=$rep', round(d['value'],4), 'pgrad', k['pgrad'], 'fwd_dense', k['fwd_dense'], 'bwd_dense', k['bwd_dense'])"
done; done; done
