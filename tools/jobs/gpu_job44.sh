#!/bin/bash
export PYTHONPATH=$PWD
for K in 4 32; do
timeout 300 python bench.py --steps 10 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j44_K${K}.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j44_K${K}.json'));print('K=$K auto', round(d['value'],4), d['loss_last'])"
done
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j44_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/j44_gpu_tests.txt
