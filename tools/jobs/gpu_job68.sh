#!/bin/bash
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_trace.py -q -p no:cacheprovider -k tool 2>&1 | tail -5
