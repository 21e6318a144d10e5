#!/bin/bash
# Graph vs Pipeline vs Hybrid (the paper's comparison) through the train tool, Reddit-shaped graph,
# 16-layer GCNII H=100, all workers in one process on the one GPU (time-sliced: bytes are exact,
# times are the sum of the workers' work, not a multi-GPU number)
export PYTHONPATH=$PWD
G=er:232965:0.0021118610741919248:1:602:41:1
mkdir -p gpurun_out/j75
for cfg in "graph --workers 4" "pipeline --stages 4" "hybrid --stages 2 --parts 2" "sequential"; do
  name=$(echo $cfg | cut -d' ' -f1)
  timeout 900 python tools/gnnpipe_train.py --synthetic $G --model gcnii --layers 16 --hidden 100 --epochs 4 \
     --compare --mode $cfg --out gpurun_out/j75/$name > gpurun_out/j75/$name.log 2>&1; echo "$name rc=$?"
  tail -2 gpurun_out/j75/$name.log
  rm -f gpurun_out/j75/$name/*.ckpt
done
timeout 600 python tools/gnnpipe_train.py --synthetic $G --model gcnii --layers 16 --hidden 100 --epochs 3 \
   --mode pipeline --stages 4 --trace --out gpurun_out/j75/pipeline_trace > gpurun_out/j75/pipeline_trace.log 2>&1; echo "trace rc=$?"
tail -2 gpurun_out/j75/pipeline_trace.log; rm -f gpurun_out/j75/pipeline_trace/*.ckpt
ls -la gpurun_out/j75/*/
