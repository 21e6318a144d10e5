#!/bin/bash
# device graph build edge cases (isolated vertices, no self loops, K = 64); parity suite; driver bench
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider > gpurun_out/j101_tests.txt 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/j101_tests.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/j101_bench.json 2> gpurun_out/j101_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j101_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['kernel_ms_per_epoch'], d['clocks'])"
