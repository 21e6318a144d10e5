#!/bin/bash
for K in 32 4; do for w in 2 3 4; do
GP_WAVE=$w timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j24_K${K}_w$w.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j24_K${K}_w$w.json'));print('K=$K wave=$w', round(d['value'],4), d['loss_last'])"
done; done
