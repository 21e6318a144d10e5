#!/bin/bash
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/j69_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/j69_gpu_tests.txt
for K in 4 32; do
timeout 300 python bench.py --steps 10 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j69_K$K.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j69_K$K.json'));print('K=$K', round(d['value'],4), d['kernel_ms_per_epoch']['bwd_agg'], d['loss_last'])"
done
