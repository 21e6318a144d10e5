#!/bin/bash
# Other BASELINE configs on one GPU: arxiv-shaped 16-layer GCN (configs[1]); products-shaped GCNII,
# 8-layer slice (= one of 8 stages of configs[3]) with the K sweep; ER-4K (configs[0]).
export PYTHONPATH=$PWD
timeout 600 python bench.py --workload arxiv --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/j47_arxiv.json 2>gpurun_out/j47_arxiv.err; python -c "import json;d=json.load(open('gpurun_out/j47_arxiv.json'));print('arxiv', d['value'], d['e2e']['value'], d['edges_per_s'])"
timeout 600 python bench.py --workload er4k --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/j47_er4k.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/j47_er4k.json'));print('er4k', d['value'], d['e2e']['value'])"
for K in 4 8 16 32; do
timeout 900 python bench.py --workload products --layers 8 --chunks $K --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j47_products_K$K.json 2>gpurun_out/j47_products_K$K.err
python -c "import json;d=json.load(open('gpurun_out/j47_products_K$K.json'));print('products 8-layer K=$K', d['value'], d['kernel_ms_per_epoch'], d['config']['l2_policy'])"
done
