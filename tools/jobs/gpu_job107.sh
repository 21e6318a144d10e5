#!/bin/bash
# transforms: A chunks in flight 3 (lib) vs 2 vs 1 at K = 32, 3 reps interleaved
export PYTHONPATH=$PWD
mkdir -p gpurun_out
P=$PWD/paper_2308_10087_b200
for rep in 1 2 3; do
for L in lib lib_xpf2 lib_xpf1; do
  GP_LIBDIR=$P/$L timeout 400 python bench.py --chunks 32 --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j107_${L}_r$rep.json 2> gpurun_out/j107_${L}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j107_${L}_r$rep.json')); print('K=32 $L rep=$rep', round(d['value'],4))"
done; done
