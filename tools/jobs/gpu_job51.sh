#!/bin/bash
export PYTHONPATH=$PWD
GP_HOST_TIMING=1 timeout 600 python tools/e2e_probe.py 2>&1 | tail -12
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j51_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/j51_gpu_tests.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/j51_bench.json 2> gpurun_out/j51_bench.err; python -c "import json;d=json.load(open('gpurun_out/j51_bench.json'));print('bench', d['value'], d['e2e']['value'])"
