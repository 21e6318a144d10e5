#!/bin/bash
# pgrad: rotated shared-store order (bank conflicts) + 4-deep prefetch; bench K = 4 / 32
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py -q -m gpu -p no:cacheprovider -x > gpurun_out/j87_tests.txt 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/j87_tests.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -k filtered_csr > gpurun_out/j87_fullsize.txt 2>&1; echo "fullsize rc=$?"; tail -2 gpurun_out/j87_fullsize.txt
for K in 4 32; do
  timeout 400 python bench.py --chunks $K --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j87_b_K${K}.json 2> gpurun_out/j87_b_K${K}.err
  python -c "import json; d=json.load(open('gpurun_out/j87_b_K${K}.json')); print('K=$K', round(d['value'],4), d['kernel_ms_per_epoch'], d['roofline']['frac'])"
done
