#!/bin/bash
# transform A-stage stride chosen by launch size (GP_XF_PAD): variants, bitwise vs lib_old, A/B
export PYTHONPATH=$PWD
mkdir -p gpurun_out
P=$PWD/paper_2308_10087_b200
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k variants > gpurun_out/j93_tests.txt 2>&1; echo "variants rc=$?"; tail -2 gpurun_out/j93_tests.txt
timeout 600 python tools/ab_bitwise.py $P/lib_old $P/lib --workload reddit > gpurun_out/j93_ab.txt 2>&1; echo "ab reddit rc=$?"; grep bitwise gpurun_out/j93_ab.txt
for rep in 1 2 3; do
for K in 32 4; do
for L in lib lib_old; do
  GP_LIBDIR=$P/$L timeout 400 python bench.py --chunks $K --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j93_b_K${K}_${L}_r$rep.json 2> gpurun_out/j93_b_K${K}_${L}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j93_b_K${K}_${L}_r$rep.json')); print('K=$K $L rep=$rep', round(d['value'],4))"
done; done; done
