"""Times the public train_pipeline call (Reddit-shaped, 64-layer GCNII) at two epoch counts to split
the per-call setup from the per-epoch cost."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2308_10087_b200 as gp
N, E2 = 232965, 114615892
ds = gp.Dataset.synthetic_er(N, E2 / (N * (N - 1)), 1, 602, 41, 1)
chunk_of = gp.make_chunks(ds, 4, 1)
model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=64, hidden=100, dropout=0.5)
for T in (1, 1, 6):
    t0 = time.perf_counter()
    res = gp.train_pipeline(ds, chunk_of, 1, gp.TrainOptions(model=model, epochs=T, seed=1, device=0))
    print(f"split={os.environ.get('GP_SPLIT', 'default')} epochs={T} wall {time.perf_counter() - t0:.3f} s", flush=True)
