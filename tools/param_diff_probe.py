"""Distribution of parameter differences vs the reference for the 16-layer / 20-epoch golden."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_10087_b200 as gp
ref = dict(np.load("tests/golden/train_gcn16_arxivlike_s2k8_20ep.npz"))
ds = gp.Dataset.synthetic_er(20000, 0.0007, 21, 128, 40, 5)
co = gp.make_chunks(ds, 8, 6)
res = gp.train_pipeline(ds, co, 2, gp.TrainOptions(model=gp.ModelConfig(kind=0, layers=16, hidden=64), epochs=20,
                                                   seed=61, fix_alpha=10))
for l, (W, b) in enumerate(res.params):
    rW = ref[f"W{l}"].astype(np.float64)
    d = np.abs(W - rW)
    rel = d / np.maximum(np.abs(rW), 1e-3)
    print(l, f"absmax {d.max():.2e} |W|max {np.abs(rW).max():.2e} rel q50 {np.quantile(rel,.5):.1e} q99 {np.quantile(rel,.99):.1e} "
          f"q999 {np.quantile(rel,.999):.1e} max {rel.max():.1e} frac>1e-3 {(rel>1e-3).mean():.1e}")

# the engine against itself with another parameter-gradient summation order (CUDA cores): the same
# amplification appears without any semantic difference
os.environ["GP_PGRAD"] = "simt"
res2 = gp.train_pipeline(ds, co, 2, gp.TrainOptions(model=gp.ModelConfig(kind=0, layers=16, hidden=64), epochs=20,
                                                    seed=61, fix_alpha=10))
print("loss rel (tc vs simt)", float(np.max(np.abs(res2.train_loss - res.train_loss) / res.train_loss)))
for l in (0, 5, 10, 14):
    d = np.abs(res2.params[l][0].astype(np.float64) - res.params[l][0])
    print("tc vs simt layer", l, f"absmax {d.max():.2e}")
