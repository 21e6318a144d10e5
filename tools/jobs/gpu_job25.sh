#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_trace.py -q -x -p no:cacheprovider 2>&1 | tail -25
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/j25_gpu_tests.txt 2>&1; tail -2 gpurun_out/j25_gpu_tests.txt
