#!/bin/bash
export PYTHONPATH=$PWD
timeout 80 python tools/ipc_same_process_probe.py 2>&1 | tail -2
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/j34_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/j34_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
