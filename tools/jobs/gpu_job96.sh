#!/bin/bash
# K = 32 with the conflict-free transform stride everywhere (GP_XF_PAD=1) vs the size rule; the
# other BASELINE shapes on the current kernels
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in 1 16384; do
  GP_XF_PAD=$v timeout 400 python bench.py --chunks 32 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j96_K32_pad${v}_r$rep.json 2> gpurun_out/j96_K32_pad${v}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j96_K32_pad${v}_r$rep.json')); k=d['kernel_ms_per_epoch']; print('K=32 pad=$v rep=$rep', round(d['value'],4), 'fwd_dense', k['fwd_dense'], 'bwd_dense', k['bwd_dense'])"
done; done
timeout 600 python bench.py --workload products --layers 8 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/j96_products8.json 2> gpurun_out/j96_products8.err; echo "products rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j96_products8.json')); print('products8', round(d['value'],4), d['e2e']['value'], d['kernel_ms_per_epoch'])"
timeout 600 python bench.py --workload arxiv --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/j96_arxiv.json 2> gpurun_out/j96_arxiv.err; echo "arxiv rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j96_arxiv.json')); print('arxiv', round(d['value'],5), d['e2e']['value'], d['config'].get('layers'), d['config'].get('stages'), d['config'].get('chunks'))"
timeout 600 python bench.py --workload er4k --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/j96_er4k.json 2> gpurun_out/j96_er4k.err; echo "er4k rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j96_er4k.json')); print('er4k', round(d['value'],5), d['e2e']['value'])"
