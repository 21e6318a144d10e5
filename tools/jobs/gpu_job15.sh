#!/bin/bash
# Split row path with the register-tiled transforms: harness timing + bit-equality, parity suite under
# GP_SPLIT=1, epoch time split vs fused at K=4 and K=32.
mkdir -p gpurun_out
./tools/fwd_bench > gpurun_out/j15_fb.txt 2>&1; grep -E "engine|split|checksum|differing" gpurun_out/j15_fb.txt
GP_SPLIT=1 timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "not ipc" > gpurun_out/j15_tests_split.txt 2>&1; tail -2 gpurun_out/j15_tests_split.txt
for K in 4 32; do for s in 0 1; do
GP_SPLIT=$s timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/j15_K${K}_s$s.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/j15_K${K}_s$s.json'));print('K=$K split=$s', round(d['value'],4), d['kernel_ms_per_epoch'], d['loss_last'])"
done; done
