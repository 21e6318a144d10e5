#!/bin/bash
# own u64 scan (replaces CUB in the filtered-CSR build): standalone check + bitwise variant tests + bench
export PYTHONPATH=$PWD
mkdir -p gpurun_out
./tools/scan_check; echo "scan_check rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -k "variants or filtered_csr" > gpurun_out/j119_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/j119_tests.txt
timeout 600 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j119_bench.json 2> gpurun_out/j119_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j119_bench.json')); print(d['value'])"
timeout 600 python bench.py --workload products --layers 8 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/j119_products8.json 2> gpurun_out/j119_products8.err; echo "products rc=$?"
python -c "import json; d=json.load(open('gpurun_out/j119_products8.json')); print('products8', round(d['value'],4), d['e2e']['value'])"
