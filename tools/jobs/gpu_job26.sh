#!/bin/bash
timeout 300 python -X faulthandler -m pytest tests/test_gpu_trace.py -q -x -p no:cacheprovider > gpurun_out/j26_trace.txt 2>&1; echo "trace rc=$?"
grep -m3 -B2 -A12 "Fatal\|Error" gpurun_out/j26_trace.txt | head -40
timeout 300 python -m pytest tests/test_gpu_ipc.py -q -x -p no:cacheprovider -k same_process > gpurun_out/j26_ipc.txt 2>&1; echo "ipc rc=$?"; tail -3 gpurun_out/j26_ipc.txt
