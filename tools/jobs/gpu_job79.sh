#!/bin/bash
# wavefront width sweep (GP_WAVE 4/6/8) at K=32 and K=8
export PYTHONPATH=$PWD
for K in 32 8; do for W in 4 6 8; do
GP_WAVE=$W timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j79_W${W}_K$K.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j79_W${W}_K$K.json'));print('W=$W K=$K', round(d['value'],4))"
done; done
