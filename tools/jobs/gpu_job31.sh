#!/bin/bash
export PYTHONPATH=$PWD
timeout 200 python -m pytest tests/test_gpu_trace.py -q -x -p no:cacheprovider > /tmp/tr.txt 2>&1; echo "trace rc=$?"; tail -3 /tmp/tr.txt
for c in 32 8; do CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 100 python -m pytest tests/test_gpu_ipc.py -q -x -p no:cacheprovider -k same_process > /tmp/ipc.txt 2>&1; echo "max_conn=$c ipc rc=$?"; tail -1 /tmp/ipc.txt; done
