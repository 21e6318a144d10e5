#!/bin/bash
# device-side graph build (k_build_edges): tests, e2e A/B with host timing
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "variants" > gpurun_out/j97_tests.txt 2>&1; echo "variants rc=$?"; tail -2 gpurun_out/j97_tests.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -k "graph" > gpurun_out/j97_fullsize.txt 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/j97_fullsize.txt
for rep in 1 2; do
for m in auto host; do
  GP_GRAPH_BUILD=$m GP_HOST_TIMING=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/j97_e2e_${m}_r$rep.json 2> gpurun_out/j97_e2e_${m}_r$rep.err
  python -c "import json; d=json.load(open('gpurun_out/j97_e2e_${m}_r$rep.json')); print('$m rep=$rep', round(d['value'],4), 'e2e', round(d['e2e']['value'],4), d['e2e']['h2d_bytes_per_step'])"
  grep "gp host" gpurun_out/j97_e2e_${m}_r$rep.err | tr '\n' ' '; echo
done; done
