#!/bin/bash
# remask with 4 rows per warp step: bitwise vs the previous build, parity, A/B
export PYTHONPATH=$PWD
mkdir -p gpurun_out
P=$PWD/paper_2308_10087_b200
timeout 600 python tools/ab_bitwise.py $P/lib_prev $P/lib --workload reddit > gpurun_out/j122_ab.txt 2>&1; echo "ab rc=$?"; grep bitwise gpurun_out/j122_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -m gpu -p no:cacheprovider > gpurun_out/j122_tests.txt 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/j122_tests.txt
for rep in 1 2; do
for L in lib lib_prev; do
  GP_LIBDIR=$P/$L timeout 400 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j122_${L}_r$rep.json 2> gpurun_out/j122_${L}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j122_${L}_r$rep.json')); print('$L rep=$rep', round(d['value'],4), 'remask', d['kernel_ms_per_epoch']['remask'])"
done; done
