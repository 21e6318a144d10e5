#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for v in 1 0 1; do
GP_FUSED_STEP=$v timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "powerlaw" > gpurun_out/j110_f$v.txt 2>&1; echo "fused=$v rc=$?"; tail -1 gpurun_out/j110_f$v.txt
done
