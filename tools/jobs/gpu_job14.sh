#!/bin/bash
# Re-entry evidence refresh: GPU parity suite, smoke, bench lines, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/j14_smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/j14_gpu_tests.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/j14_gpu_tests.txt
tail -3 gpurun_out/j14_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j14_smoke.txt 2>&1; tail -2 gpurun_out/j14_smoke.txt
timeout 900 python bench.py > gpurun_out/j14_bench.json 2> gpurun_out/j14_bench.err; tail -c 600 gpurun_out/j14_bench.json
timeout 400 python bench.py --steps 5 --warmup 3 --chunks 32 --no-e2e --no-cpu-baseline > gpurun_out/j14_K32.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j14_K32.json'));print('K=32', round(d['value'],4), d['kernel_ms_per_epoch'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/j14_ref.json 2>gpurun_out/j14_ref.err; tail -c 300 gpurun_out/j14_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j14_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j14_ncu_bench.log 2>&1; echo "ncu rc=$?"
