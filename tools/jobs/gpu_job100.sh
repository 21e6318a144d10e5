#!/bin/bash
# e2e diagnosis: the driver's command with GP_HOST_TIMING, twice
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for rep in 1 2; do
GP_HOST_TIMING=1 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/j100_bench_r$rep.json 2> gpurun_out/j100_bench_r$rep.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j100_bench_r$rep.json')); print(d['value'], d['e2e']['value'])"
grep "gp host\|gp graph\|gp upload" gpurun_out/j100_bench_r$rep.err | tail -14 | tr -s ' ' | tr '\n' ';'; echo
grep "gp epoch" gpurun_out/j100_bench_r$rep.err | tail -22 | awk '{print $5, $7, $9}' | tr '\n' ';'; echo
done
