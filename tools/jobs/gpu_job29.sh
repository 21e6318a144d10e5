#!/bin/bash
export PYTHONPATH=$PWD
for w in 2 1 4; do GP_WAVE=$w timeout 100 python -m pytest tests/test_gpu_ipc.py -q -x -p no:cacheprovider -k same_process > /tmp/ipc_$w.txt 2>&1; echo "wave=$w ipc rc=$?"; tail -1 /tmp/ipc_$w.txt; done
timeout 200 python -X faulthandler -m pytest tests/test_gpu_trace.py -q -x -p no:cacheprovider > /tmp/tr.txt 2>&1; echo "trace rc=$?"; grep -E "passed|failed|Fatal|Error" /tmp/tr.txt | head -5
