#!/bin/bash
# Final round-1 check on a fresh box: GPU suite, smoke, default bench, reference arm (driver's commands).
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/j48_gpu_tests.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/j48_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/j48_bench.json 2> gpurun_out/j48_bench.err; python -c "import json;d=json.load(open('gpurun_out/j48_bench.json'));print('bench', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['gather_frac'], d['gpu_launches'], d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/j48_ref.json 2> gpurun_out/j48_ref.err; python -c "import json;d=json.load(open('gpurun_out/j48_ref.json'));print('ref', d['value'], d['cpu_baseline']['sample'][:80])"
