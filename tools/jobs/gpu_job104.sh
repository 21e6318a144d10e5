#!/bin/bash
# drop-in C++ callers rebuilt against the updated header
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dropin.py -q -m gpu -p no:cacheprovider > gpurun_out/j104_dropin.txt 2>&1; echo "dropin rc=$?"; tail -2 gpurun_out/j104_dropin.txt
