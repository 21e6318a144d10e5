set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
ncu --set full --clock-control none --import-source on -k regex:"k_fwd8|k_bwd8|k_pgrad_partial|k_dense_gemm" -s 10 -c 6 -o gpurun_out/prof_r1c python bench.py --layers 6 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r1c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/launch_r1c.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
nproc > gpurun_out/nproc.txt; lscpu | head -20 > gpurun_out/lscpu.txt
