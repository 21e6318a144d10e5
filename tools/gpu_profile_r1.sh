# Round-1 evidence: bench lines, launch list, ncu --set full of the dominant kernel.
set -x
nvidia-smi -L
timeout 900 python bench.py > gpurun_out/p_bench_n1.json 2> gpurun_out/p_bench_n1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/p_bench_ref.json 2> gpurun_out/p_bench_ref.err
# launch list: 3 warm-up epochs skipped approximately; 1 timed + the profiling epoch captured
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p_launch_bench.json 2> gpurun_out/p_launch.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fwd8 -s 40 -c 1 -o gpurun_out/p_fwd8 \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/p_ncu_fwd.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bwd8 -s 40 -c 1 -o gpurun_out/p_bwd8 \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/p_ncu_bwd.err
ls -la gpurun_out/
