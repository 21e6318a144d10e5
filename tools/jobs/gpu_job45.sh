#!/bin/bash
export PYTHONPATH=$PWD
GP_HOST_TIMING=1 timeout 600 python tools/e2e_probe.py 2>&1 | grep -E "gp_create|destroy|wall"
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j45_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/j45_gpu_tests.txt
timeout 900 python bench.py > gpurun_out/j45_bench.json 2> gpurun_out/j45_bench.err; python -c "import json;d=json.load(open('gpurun_out/j45_bench.json'));print(d['value'], d['e2e'])"
