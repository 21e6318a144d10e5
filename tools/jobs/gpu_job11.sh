timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.txt 2>&1; tail -2 gpurun_out/gpu_all.txt; grep -E "FAILED|Error" gpurun_out/gpu_all.txt | head -5
for K in 4 32; do for w in 1 0; do
GP_WAVE=$w timeout 300 python bench.py --steps 5 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/b11_K${K}_w$w.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b11_K${K}_w$w.json'));print('K=$K wave=$w', round(d['value'],4), d['kernel_ms_per_epoch'], d['loss_last'])"
done; done
./tools/fwd_bench 2>&1 | grep -E "engine|split|checksum"
