#!/bin/bash
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j62_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/j62_gpu_tests.txt
GP_SPLIT=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/j62_fused.txt 2>&1; echo "fused rc=$?"; tail -1 gpurun_out/j62_fused.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
