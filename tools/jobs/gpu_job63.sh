#!/bin/bash
export PYTHONPATH=$PWD
for tr in 4 2 1; do
GP_TILE_TR=$tr timeout 300 python bench.py --steps 5 --warmup 3 --chunks 32 --no-e2e --no-cpu-baseline > gpurun_out/j63_tr$tr.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j63_tr$tr.json'));k=d['kernel_ms_per_epoch'];print('K=32 TR=$tr', round(d['value'],4), k['fwd_dense'], k['bwd_dense'])"
done
