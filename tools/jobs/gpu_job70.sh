#!/bin/bash
export PYTHONPATH=$PWD
for K in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j70_K$K.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j70_K$K.json'));print('K=$K', round(d['value'],4), d['kernel_ms_per_epoch'])"
done
