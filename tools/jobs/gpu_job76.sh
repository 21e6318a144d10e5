#!/bin/bash
# gathers in flight: GP_NB=4 (split kernels, 4 CTAs/SM) vs default, K=4 and K=32
export PYTHONPATH=$PWD
for NB in 2 4; do for K in 4 32; do
GP_NB=$NB timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j76_NB${NB}_K$K.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j76_NB${NB}_K$K.json'));print('NB=$NB K=$K', round(d['value'],4), d['kernel_ms_per_epoch']['fwd_agg'], d['kernel_ms_per_epoch']['bwd_agg'])"
done; done
