#!/bin/bash
echo "== v3 (a0338a0) same-process"; PYTHONPATH=$PWD/variants/v3:$PWD timeout 100 python -m pytest tests/test_gpu_ipc.py -q -x -p no:cacheprovider -k same_process > /tmp/v3.txt 2>&1; echo rc=$?; tail -1 /tmp/v3.txt
export PYTHONPATH=$PWD
echo "== current, cross-process"; timeout 400 python -m pytest tests/test_gpu_ipc.py -q -p no:cacheprovider -k "not same_process" > /tmp/xp.txt 2>&1; echo rc=$?; tail -3 /tmp/xp.txt
nvidia-smi --query-gpu=name,driver_version,clocks.sm --format=csv
