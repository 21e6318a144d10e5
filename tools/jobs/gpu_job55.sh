#!/bin/bash
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "sage or invalid" 2>&1 | tail -15
