#!/bin/bash
# K = 32 with the padded-stride transforms: wavefront width sweep (lib) vs lib_old at its default
export PYTHONPATH=$PWD
mkdir -p gpurun_out
P=$PWD/paper_2308_10087_b200
for rep in 1 2; do
for cfg in "lib 12" "lib 8" "lib 6" "lib 16" "lib_old 12" "lib_old 8"; do
  set -- $cfg
  GP_LIBDIR=$P/$1 GP_WAVE=$2 timeout 400 python bench.py --chunks 32 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j92_$1_w$2_r$rep.json 2> gpurun_out/j92_$1_w$2_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j92_$1_w$2_r$rep.json')); print('$1 W=$2 rep=$rep', round(d['value'],4))"
done; done
