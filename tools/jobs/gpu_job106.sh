#!/bin/bash
# tcgen05 transforms: A chunks in flight 2 (lib) vs 1 (lib_xpf1, the previous loop) vs 3 (lib_xpf3)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
P=$PWD/paper_2308_10087_b200
timeout 600 python tools/ab_bitwise.py $P/lib_xpf1 $P/lib --workload reddit > gpurun_out/j106_ab.txt 2>&1; echo "ab rc=$?"; grep bitwise gpurun_out/j106_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x > gpurun_out/j106_tests.txt 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/j106_tests.txt
for rep in 1 2; do
for K in 4 32; do
for L in lib lib_xpf1 lib_xpf3; do
  GP_LIBDIR=$P/$L timeout 400 python bench.py --chunks $K --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j106_K${K}_${L}_r$rep.json 2> gpurun_out/j106_K${K}_${L}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j106_K${K}_${L}_r$rep.json')); k=d['kernel_ms_per_epoch']; print('K=$K $L rep=$rep', round(d['value'],4), 'fwd_dense', k['fwd_dense'], 'bwd_dense', k['bwd_dense'])"
done; done; done
