#!/bin/bash
# done-filtered backward CSR (GP_BWD_CSR): bitwise variants + A/B epoch time at K = 4 and K = 32
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "variants" tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider > gpurun_out/j85_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/j85_tests.txt
for rep in 1 2; do
for K in 4 32; do
for v in 1 0; do
  GP_BWD_CSR=$v timeout 400 python bench.py --chunks $K --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j85_b_K${K}_csr${v}_r$rep.json 2> gpurun_out/j85_b_K${K}_csr${v}_r$rep.err
  python -c "import json,sys; d=json.load(open('gpurun_out/j85_b_K${K}_csr${v}_r$rep.json')); print('K=$K csr=$v rep=$rep', round(d['value'],4), d['kernel_ms_per_epoch'].get('bwd_agg'), d['kernel_span_ms_per_epoch'].get('bwd_agg'))"
done; done; done
