#!/bin/bash
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider 2>&1 | tail -15
