#!/bin/bash
# remask overlap (GP_REMASK_OVERLAP): bitwise variants, full-size wavefront tests, A/B at K = 4 and 32
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k variants > gpurun_out/j89_tests.txt 2>&1; echo "variants rc=$?"; tail -2 gpurun_out/j89_tests.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider > gpurun_out/j89_fullsize.txt 2>&1; echo "fullsize rc=$?"; tail -2 gpurun_out/j89_fullsize.txt
for rep in 1 2; do
for K in 4 32; do
for v in 1 0; do
  GP_REMASK_OVERLAP=$v timeout 400 python bench.py --chunks $K --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j89_b_K${K}_ovl${v}_r$rep.json 2> gpurun_out/j89_b_K${K}_ovl${v}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j89_b_K${K}_ovl${v}_r$rep.json')); print('K=$K ovl=$v rep=$rep', round(d['value'],4), d['kernel_span_ms_per_epoch'])"
done; done; done
