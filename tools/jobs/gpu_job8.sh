./tools/fwd_bench > gpurun_out/fb_split.txt 2>&1; grep -E "engine|split|k_bwd8|checksum" gpurun_out/fb_split.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.txt 2>&1; tail -3 gpurun_out/gpu_all.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b8_split.json 2>/dev/null
GP_SPLIT=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b8_fused.json 2>/dev/null
timeout 300 python bench.py --steps 3 --warmup 3 --chunks 32 --no-e2e --no-cpu-baseline > gpurun_out/b8_split_k32.json 2>/dev/null
for f in b8_split b8_fused b8_split_k32; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['value'],4), d['kernel_ms_per_epoch'], d['loss_last'])"; done
