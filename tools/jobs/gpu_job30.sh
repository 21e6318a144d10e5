#!/bin/bash
export PYTHONPATH=$PWD
LD_PRELOAD=$PWD/tools/segv_bt.so timeout 200 python -m pytest tests/test_gpu_trace.py -q -x -p no:cacheprovider -p no:faulthandler > /tmp/tr.txt 2>&1; echo "trace rc=$?"; tail -5 /tmp/tr.txt; cat /tmp/segv_bt.txt
