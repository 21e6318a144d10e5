#!/bin/bash
# Round-1 final evidence: bench lines (N=1 default, K=32, reference arm), launch list, 2-rank functional run.
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/j40_bench.json 2> gpurun_out/j40_bench.err; tail -c 300 gpurun_out/j40_bench.json; echo
timeout 600 python bench.py --steps 5 --warmup 3 --chunks 32 --no-e2e --no-cpu-baseline > gpurun_out/j40_K32.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/j40_ref.json 2>gpurun_out/j40_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j40_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launch list rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/j40_n2.json 2> gpurun_out/j40_n2.err; echo "n2 rc=$?"; tail -c 400 gpurun_out/j40_n2.json
