#!/bin/bash
# e2e phase breakdown after the GPU suite (the driver's round-end order)
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j74_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/j74_gpu_tests.txt
free -g | head -2
for r in 1 2; do
GP_HOST_TIMING=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/j74_bench$r.json 2> gpurun_out/j74_bench$r.err
python -c "import json;d=json.load(open('gpurun_out/j74_bench$r.json'));print('bench', d['value'], d['e2e']['value'], d['host_prep_s'])"
grep "gp host" gpurun_out/j74_bench$r.err
done
