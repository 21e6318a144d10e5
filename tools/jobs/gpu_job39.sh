#!/bin/bash
export PYTHONPATH=$PWD
GP_HOST_TIMING=1 timeout 600 python tools/e2e_probe.py 2>&1 | grep -E "gp_create|graph|create\+upload|destroy|wall"
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j39_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/j39_gpu_tests.txt
