#!/bin/bash
# two-ahead CSR-entry prefetch in the done-filtered gather: bench K=4/K=32 + backward parity subset
export PYTHONPATH=$PWD
for K in 4 32; do
timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j78_K$K.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j78_K$K.json'));print('PF2 K=$K', round(d['value'],4), d['kernel_ms_per_epoch']['fwd_agg'], d['kernel_ms_per_epoch']['bwd_agg'])"
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider 2>&1 | tail -2
