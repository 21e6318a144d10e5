#!/bin/bash
# evidence on the current code: GPU suite, smoke, driver-command bench, launch list, ncu --set full of
# the backward gather (pre-filtered CSR), the filter-CSR build and the transforms
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j94_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j94_gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/j94_gpu_tests.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/j94_bench.json 2> gpurun_out/j94_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j94_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/j94_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/j94_ncu_list.log 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/j94_launches.csv "# ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 python bench.py --steps 1 --warmup 1 (current kernels: pre-filtered backward CSR, remask overlap, padded transform staging)" > gpurun_out/j94_launches_summary.txt; head -20 gpurun_out/j94_launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_bwd8<6," --launch-skip 24 -c 4 -f -o gpurun_out/j94_ncu_bwd python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu bwd rc=$?"
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:k_done_csr" -c 2 -f -o gpurun_out/j94_ncu_donecsr python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu donecsr rc=$?"
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:k_tc_xform" --launch-skip 40 -c 4 -f -o gpurun_out/j94_ncu_xform python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu xform rc=$?"
for r in bwd donecsr xform; do
  ncu -i gpurun_out/j94_ncu_$r.ncu-rep --page details --csv > gpurun_out/j94_ncu_${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/j94_ncu_$r.ncu-rep --page raw --csv > gpurun_out/j94_ncu_${r}_raw.csv 2>/dev/null
  rm -f gpurun_out/j94_ncu_$r.ncu-rep
done
ls -la gpurun_out/ | grep j94
