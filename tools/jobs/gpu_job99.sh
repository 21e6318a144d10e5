#!/bin/bash
# final evidence of the session: GPU suite, smoke, driver-command bench, K = 32 bench, sanitizer on the new kernels
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j99_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j99_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/j99_gpu_tests.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/j99_bench.json 2> gpurun_out/j99_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j99_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['gather_frac_span'], d['epoch_gather_bound']['frac'], d['clocks'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --chunks 32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/j99_bench_k32.json 2> gpurun_out/j99_bench_k32.err; echo "bench k32 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j99_bench_k32.json')); print(d['value'], d['e2e']['value'])"
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "variants and (device_graph_build or batch_filter or remask_in_order or xf_dense or one_stream)" > gpurun_out/j99_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/j99_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j99_racecheck_smoke.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/j99_racecheck_smoke.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "variants and device_graph_build and pipeline and stale" > gpurun_out/j99_racecheck_new.txt 2>&1; echo "racecheck new rc=$?"; tail -3 gpurun_out/j99_racecheck_new.txt
