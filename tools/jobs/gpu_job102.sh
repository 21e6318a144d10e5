#!/bin/bash
# proxy for a layer-major S = 1 schedule: K = 1 (one launch per layer over all rows, one table)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for K in 1 4; do
timeout 600 python bench.py --chunks $K --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j102_K$K.json 2> gpurun_out/j102_K$K.err; echo "K=$K rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j102_K$K.json')); print(round(d['value'],4), d['kernel_ms_per_epoch'], d['kernel_span_ms_per_epoch'], d['gather_frac_span'], d['roofline']['gather_frac_serial'])"
done
