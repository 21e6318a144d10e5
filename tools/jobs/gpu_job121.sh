#!/bin/bash
# K = 32 wavefront width with the session's final kernels
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for rep in 1 2 3; do
for w in 12 16 8; do
  GP_WAVE=$w timeout 400 python bench.py --chunks 32 --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j121_w${w}_r$rep.json 2> gpurun_out/j121_w${w}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j121_w${w}_r$rep.json')); print('K=32 W=$w rep=$rep', round(d['value'],4))"
done; done
