#!/bin/bash
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j69_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/j69_gpu_tests.txt
