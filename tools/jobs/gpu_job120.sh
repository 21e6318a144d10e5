#!/bin/bash
# final code of the session (own scan): smoke, GPU suite, driver-command bench, K = 32 bench
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j120_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/j120_smoke.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j120_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/j120_gpu_tests.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/j120_bench.json 2> gpurun_out/j120_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j120_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['gather_frac_span'], d['epoch_gather_bound']['frac'], d['clocks'], d['cpu_baseline']['value'], d['kernel_ms_per_epoch'])"
timeout 900 python bench.py --chunks 32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/j120_bench_k32.json 2> gpurun_out/j120_bench_k32.err; echo "bench k32 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j120_bench_k32.json')); print(d['value'], d['e2e']['value'])"
