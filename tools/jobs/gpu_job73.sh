#!/bin/bash
# e2e phase breakdown (GP_HOST_TIMING) on the headline config
export PYTHONPATH=$PWD
nproc; lscpu | grep -i "model name"
GP_HOST_TIMING=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/j73_bench.json 2> gpurun_out/j73_bench.err
python -c "import json;d=json.load(open('gpurun_out/j73_bench.json'));print('bench', d['value'], d['e2e']['value'], d['host_prep_s'])"
grep -v "^\s*$" gpurun_out/j73_bench.err | tail -25
