#!/bin/bash
# fresh-container rebuild: GPU suite + default bench (driver command) + smoke
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j84_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j84_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/j84_gpu_tests.txt
timeout 600 python bench.py > gpurun_out/j84_bench.json 2> gpurun_out/j84_bench.err; echo "bench rc=$?"; cat gpurun_out/j84_bench.json | head -c 600
