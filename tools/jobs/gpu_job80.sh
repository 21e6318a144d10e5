#!/bin/bash
# HEAD check: GPU suite + smoke
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j80_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/j80_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
