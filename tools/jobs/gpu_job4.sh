set -x
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_ipc.py -q -m gpu -x > gpurun_out/gpu_ipc.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.txt 2>&1
tail -3 gpurun_out/gpu_ipc.txt gpurun_out/gpu_all.txt; cat gpurun_out/bench_n2_shared.json; tail -5 gpurun_out/bench_n2_shared.err
