"""Determinism probe: train the same configuration R times in fresh processes under one engine
setting and report whether every run is bit-identical to the first.

    python tools/det_probe.py '<json config>' R [ENV=VAL ...]"""
import json
import os
import subprocess
import sys

import numpy as np

CHILD = r'''
import sys, json, numpy as np, os
sys.path.insert(0, os.getcwd())
import paper_2308_10087_b200 as gp
cfg = json.loads(sys.argv[1])
if cfg["data"] == "powerlaw":
    ds = gp.Dataset.load("tests/golden/powerlaw_2k")
else:
    ds = gp.Dataset.synthetic_er(500, 0.02, 3, cfg.get("F", 16), cfg.get("C", 5), 9)
co = gp.make_chunks(ds, cfg["K"], cfg.get("cs", 4))
opt = gp.TrainOptions(model=gp.ModelConfig(kind=cfg["kind"], layers=cfg["L"], hidden=16), epochs=cfg["ep"],
                      seed=cfg.get("seed", 51), fix_alpha=cfg.get("fa", 3))
if cfg["G"] > 1:
    part, _, _ = gp.partition_vertices(ds, cfg["G"], cfg.get("ps", 1))
    r = gp.train_hybrid(ds, part, co, cfg["S"], opt)
else:
    r = gp.train_pipeline(ds, co, cfg["S"], opt)
np.save(sys.argv[2], np.concatenate([r.train_loss.astype(np.float64)] + [w.ravel().astype(np.float64) for w, b in r.params]))
'''


def main():
    cfg, reps = sys.argv[1], int(sys.argv[2])
    env = dict(os.environ)
    for kv in sys.argv[3:]:
        k, v = kv.split("=", 1)
        env[k] = v
    outs = []
    for i in range(reps):
        subprocess.run([sys.executable, "-c", CHILD, cfg, f"/tmp/det_{i}.npy"], env=env, check=True)
        outs.append(np.load(f"/tmp/det_{i}.npy"))
    same = [np.array_equal(outs[0], o) for o in outs]
    print(cfg, sys.argv[3:], "deterministic" if all(same) else f"NONDETERMINISTIC {same}", flush=True)


if __name__ == "__main__":
    main()
