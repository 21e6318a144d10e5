#!/bin/bash
# merged gather tables (GP_MERGED_G=1): parity suite + bench K=4 / K=32 against the split tables
export PYTHONPATH=$PWD
GP_MERGED_G=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/j71_tests_merged.txt 2>&1; echo "merged tests rc=$?"; tail -3 gpurun_out/j71_tests_merged.txt
for M in 0 1; do for K in 4 32; do
GP_MERGED_G=$M timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j71_M${M}_K$K.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j71_M${M}_K$K.json'));print('M=$M K=$K', round(d['value'],4), d['kernel_ms_per_epoch'])"
done; done
