#!/bin/bash
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "grads or adam or variants or wide" 2>&1 | tail -5
for m in tc1 tc; do
GP_PGRAD=$m timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j64_$m.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j64_$m.json'));print('$m', round(d['value'],4), d['kernel_ms_per_epoch']['pgrad'], d['loss_last'])"
done
GP_PGRAD=tc timeout 300 python bench.py --workload products --layers 8 --chunks 4 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/j64_prod.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/j64_prod.json'));print('products', round(d['value'],4), d['kernel_ms_per_epoch']['pgrad'])"
