#!/bin/bash
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "invalid" 2>&1 | tail -3
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j37_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/j37_gpu_tests.txt
