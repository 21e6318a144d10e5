#!/bin/bash
export PYTHONPATH=$PWD
for K in 4 32; do
timeout 900 python bench.py --workload products --layers 8 --chunks $K --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j52_products_K$K.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j52_products_K$K.json'));print('products 8-layer K=$K', d['value'], d['kernel_ms_per_epoch'])"
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j52_reddit.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/j52_reddit.json'));print('reddit', d['value'])"
