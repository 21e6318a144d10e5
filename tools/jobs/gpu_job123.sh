#!/bin/bash
# very last code: smoke + full GPU suite
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j123_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/j123_smoke.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j123_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/j123_gpu_tests.txt
