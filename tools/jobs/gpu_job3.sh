timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/gpu_tests3.txt 2>&1
for nb in 2 4; do GP_NB=$nb timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench3_nb$nb.json 2>gpurun_out/bench3_nb$nb.err; done
GP_PGRAD=simt GP_NB=2 timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench3_simt.json 2>/dev/null
