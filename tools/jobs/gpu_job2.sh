./tools/l2_gather_bench_v8 > gpurun_out/l2bench_v8.txt 2>&1
for nb in 2 4 6 8; do GP_NB=$nb python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_nb$nb.json 2>/dev/null; done
python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/gpu_tests.txt 2>&1
