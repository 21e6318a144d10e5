#!/bin/bash
# K sweep for the headline config at N=1, and the 8-stage pipeline as 8 processes on the one GPU
# (functional: the stages time-slice the device, so this is not a scaling number).
export PYTHONPATH=$PWD
for K in 8 16; do
timeout 600 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j53_K$K.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j53_K$K.json'));print('K=$K', d['value'])"
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 8 --steps 3 --warmup 3 --no-e2e > gpurun_out/j53_n8.json 2> gpurun_out/j53_n8.err; echo "n8 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/j53_n8.json'));print('8 stages on 1 GPU', d['value'], d['config']['chunks'], d['config']['ranks_per_gpu'], d['gpu_launches'], d['loss_last'])"
