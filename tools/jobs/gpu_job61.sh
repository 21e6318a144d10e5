#!/bin/bash
# One stage's share of the 8-stage Reddit pipeline on one GPU: an 8-layer GCNII (stage 0 holds the
# 602->100 Dense layer + 7 convs; a middle stage 8 convs) at K = 32 chunks.
export PYTHONPATH=$PWD
timeout 600 python bench.py --layers 8 --chunks 32 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j61_reddit_8layer_K32.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j61_reddit_8layer_K32.json'));print('reddit 8-layer K=32', d['value'], d['kernel_ms_per_epoch'])"
