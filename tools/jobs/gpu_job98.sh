#!/bin/bash
# e2e phases of the graph upload, device vs host builder (GP_HOST_TIMING), 3 reps
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for rep in 1 2 3; do
for m in auto host; do
  GP_GRAPH_BUILD=$m GP_HOST_TIMING=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/j98_e2e_${m}_r$rep.json 2> gpurun_out/j98_e2e_${m}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j98_e2e_${m}_r$rep.json')); print('$m rep=$rep', round(d['value'],4), 'e2e', round(d['e2e']['value'],4))"
  grep "gp host\|gp graph\|gp upload" gpurun_out/j98_e2e_${m}_r$rep.err | tail -16 | tr -s ' ' | tr '\n' ';'; echo
done; done
