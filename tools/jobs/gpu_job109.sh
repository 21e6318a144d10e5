#!/bin/bash
# fused optimizer step (k_param_step): parity suite + A/B
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider > gpurun_out/j109_tests.txt 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/j109_tests.txt
for rep in 1 2; do
for v in 1 0; do
  GP_FUSED_STEP=$v timeout 400 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j109_f${v}_r$rep.json 2> gpurun_out/j109_f${v}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j109_f${v}_r$rep.json')); print('fused=$v rep=$rep', round(d['value'],4), 'optim', d['kernel_ms_per_epoch']['optim'], 'launches/epoch', d['gpu_launches']//8)"
done; done
