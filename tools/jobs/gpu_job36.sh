#!/bin/bash
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "sage" 2>&1 | tail -30
