for K in 4 16 32; do for nb in 2 4 8; do
GP_NB=$nb timeout 300 python bench.py --steps 3 --warmup 3 --chunks $K --no-e2e --no-cpu-baseline > gpurun_out/b6_K${K}_nb$nb.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b6_K${K}_nb$nb.json'));print('K=$K nb=$nb', round(d['value'],4), d['kernel_ms_per_epoch'])"
done; done
