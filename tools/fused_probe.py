import os, sys, subprocess, numpy as np, json
CHILD = r'''
import sys, json, numpy as np, os
sys.path.insert(0, os.getcwd())
import paper_2308_10087_b200 as gp
cfg = json.loads(sys.argv[1])
if cfg["data"] == "powerlaw":
    ds = gp.Dataset.load("tests/golden/powerlaw_2k")
else:
    ds = gp.Dataset.synthetic_er(500, 0.02, 3, cfg.get("F", 16), cfg.get("C", 5), 9)
co = gp.make_chunks(ds, cfg["K"], 4)
opt = gp.TrainOptions(model=gp.ModelConfig(kind=cfg["kind"], layers=cfg["L"], hidden=16), epochs=cfg["ep"], seed=51, fix_alpha=3)
if cfg["G"] > 1:
    part, _, _ = gp.partition_vertices(ds, cfg["G"], 1)
    r = gp.train_hybrid(ds, part, co, cfg["S"], opt)
else:
    r = gp.train_pipeline(ds, co, cfg["S"], opt)
np.save(sys.argv[2], np.concatenate([r.train_loss.astype(np.float64)] + [w.ravel().astype(np.float64) for w, b in r.params]))
'''
cases = [dict(data="powerlaw", kind=2, L=8, S=2, G=1, K=8, ep=4), dict(data="powerlaw", kind=2, L=8, S=2, G=1, K=8, ep=4, W="1"),
         dict(data="powerlaw", kind=2, L=8, S=1, G=1, K=8, ep=4), dict(data="er", kind=2, L=8, S=2, G=1, K=8, ep=4),
         dict(data="powerlaw", kind=2, L=8, S=2, G=1, K=8, ep=4, R="0"), dict(data="powerlaw", kind=2, L=8, S=2, G=1, K=8, ep=2)]
for c in cases:
    out = {}
    for v in ("1", "0"):
        env = dict(os.environ, GP_FUSED_STEP=v)
        if "W" in c: env["GP_WAVE"] = c["W"]
        if "R" in c: env["GP_REMASK_OVERLAP"] = c["R"]
        subprocess.run([sys.executable, "-c", CHILD, json.dumps(c), f"/tmp/fp_{v}.npy"], env=env, check=True)
        out[v] = np.load(f"/tmp/fp_{v}.npy")
    print(c, "equal" if np.array_equal(out["1"], out["0"]) else f"DIFF max {np.max(np.abs(out['1'] - out['0'])):.3g}", flush=True)
