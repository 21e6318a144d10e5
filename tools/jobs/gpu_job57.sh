#!/bin/bash
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_trace.py -q -p no:cacheprovider 2>&1 | tail -15
