#!/bin/bash
# pgrad: rotated shared-store order with predicated selects; prefetch depth 4 (lib) vs 2 (lib_pf2)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "pgrad or train_gcn or variants" > gpurun_out/j88_tests.txt 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/j88_tests.txt
for rep in 1 2; do
for L in lib lib_pf2; do
  GP_LIBDIR=$PWD/paper_2308_10087_b200/$L timeout 400 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j88_b_${L}_$rep.json 2> gpurun_out/j88_b_${L}_$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j88_b_${L}_$rep.json')); print('$L', round(d['value'],4), 'pgrad', d['kernel_ms_per_epoch']['pgrad'])"
done; done
