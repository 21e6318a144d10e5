"""Per-phase wall times of one StageEngine lifecycle (Reddit shape, 64-layer GCNII, K=4)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2308_10087_b200 as gp
N, E2, F, C, H, L, K = 232965, 114615892, 602, 41, 100, 64, 4
ds = gp.Dataset.synthetic_er(N, E2 / (N * (N - 1)), 1, F, C, 1)
chunk_of = gp.make_chunks(ds, K, 1)
model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=L, hidden=H, dropout=0.5)
specs = gp.build_layer_specs(model, F, C)
params = gp.init_params(model, F, C, 1)
off, cols, vals = ds.normalize_adjacency(True)
x, lab, sp = ds.arrays()
for rep in range(2):
    T = [time.perf_counter()]
    def mark(name):
        T.append(time.perf_counter()); print(f"  {name:14s} {T[-1] - T[-2]:.3f} s", flush=True)
    eng = gp.StageEngine(num_vertices=N, num_chunks=K, specs=specs, stage=0, num_stages=1, layer_range=(0, L),
                         hidden=H, num_classes=C, dropout=0.5, seed=1, device=0)
    mark("create")
    eng.upload_graph(off, cols, vals, chunk_of); eng.synchronize(); mark("upload_graph")
    eng.upload_features(x); eng.upload_labels(lab, sp); eng.synchronize(); mark("features")
    for l in range(L):
        eng.set_params(l, *params[l])
    eng.synchronize(); mark("set_params")
    for t in range(1, 4):
        eng.run_epoch(t, gp.shuffle_chunk_order(K, t, 1)); eng.synchronize(); mark(f"epoch {t}")
    eng.close(); mark("close")
