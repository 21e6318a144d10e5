#!/bin/bash
# the driver's two arms on the last commit: reference arm then ours
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/j124_ref.json 2> gpurun_out/j124_ref.err; echo "ref rc=$?"; head -c 400 gpurun_out/j124_ref.json; echo
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/j124_bench.json 2> gpurun_out/j124_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j124_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
