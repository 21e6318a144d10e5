#!/bin/bash
export PYTHONPATH=$PWD
for K in 4 32; do for o in 0 1; do
GP_OCC5=$o timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j43_K${K}_o$o.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j43_K${K}_o$o.json'));print('K=$K occ5=$o', round(d['value'],4), d['kernel_ms_per_epoch'], d['loss_last'])"
done; done
