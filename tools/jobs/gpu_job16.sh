#!/bin/bash
mkdir -p gpurun_out
./tools/fwd_bench > gpurun_out/j16_fb.txt 2>&1; grep -E "tile|differing|K=.*engine|split gather k_fwd8<GCN2,2" gpurun_out/j16_fb.txt
for K in 4 32; do for s in 1; do
GP_SPLIT=$s timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j16_K${K}_s$s.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j16_K${K}_s$s.json'));print('K=$K split=$s', round(d['value'],4), d['kernel_ms_per_epoch'], d['loss_last'])"
done; done
