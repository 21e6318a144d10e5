#!/bin/bash
cat > /tmp/seg_probe.py <<'PY'
import sys, numpy as np
import paper_2308_10087_b200 as gp
ds = gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)
model = gp.ModelConfig(kind=gp.ModelKind.GCN, layers=6, hidden=16)
co = gp.make_chunks(ds, 4, 3)
r = gp.train_pipeline(ds, co, 2, gp.TrainOptions(model=model, epochs=3, seed=5, fix_alpha=2))
print("ok", r.train_loss, flush=True)
PY
export PYTHONPATH=$PWD
for w in 1 4; do echo "== current, GP_WAVE=$w"; GP_WAVE=$w timeout 60 python /tmp/seg_probe.py 2>&1 | tail -1
GP_WAVE=$w timeout 100 python -m pytest tests/test_gpu_ipc.py -q -x -p no:cacheprovider -k same_process 2>&1 | tail -1; done
echo "== v1 ipc"; PYTHONPATH=$PWD/variants/v1:$PWD timeout 100 python -m pytest tests/test_gpu_ipc.py -q -x -p no:cacheprovider -k same_process > /tmp/v1ipc.txt 2>&1; echo rc=$?; tail -1 /tmp/v1ipc.txt
