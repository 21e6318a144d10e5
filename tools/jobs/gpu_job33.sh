#!/bin/bash
export PYTHONPATH=$PWD
for v in "GP_IPC_SMCOPY=1" "GP_IPC_SMCOPY=1 CUDA_DEVICE_MAX_CONNECTIONS=32" "GP_WAVE=1 GP_IPC_SMCOPY=1"; do env $v timeout 100 python -m pytest tests/test_gpu_ipc.py -q -x -p no:cacheprovider -k same_process > /tmp/ipc.txt 2>&1; echo "$v ipc rc=$?"; tail -1 /tmp/ipc.txt; done
