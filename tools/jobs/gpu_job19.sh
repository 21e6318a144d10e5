#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/j19_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/j19_gpu_tests.txt; tail -3 gpurun_out/j19_gpu_tests.txt
GP_SPLIT=0 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/j19_gpu_tests_fused.txt 2>&1; tail -1 gpurun_out/j19_gpu_tests_fused.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
