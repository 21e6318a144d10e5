"""Train the same configuration with two builds of the engine (GP_LIBDIR) and report whether
losses and parameters agree bit for bit. Used to check that kernel changes which must not
alter arithmetic (layouts, scheduling) really do not.

    python tools/ab_bitwise.py <libdir_a> <libdir_b> [--workload er|reddit]
"""
import os
import subprocess
import sys

import numpy as np

CHILD = r'''
import sys, numpy as np
import paper_2308_10087_b200 as gp
w = sys.argv[1]
if w == "reddit":
    N, F, C = 232965, 602, 41
    ds = gp.Dataset.synthetic_er(N, 114615892 / (N * (N - 1)), 1, F, C, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=8, hidden=100, dropout=0.5)
    K = 4
else:
    ds = gp.Dataset.synthetic_er(4096, 0.0039, 1, 128, 16, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=8, hidden=128, dropout=0.5)
    K = 4
co = gp.make_chunks(ds, K, 1)
r = gp.train_pipeline(ds, co, 1, gp.TrainOptions(model=model, epochs=3, seed=1))
out = {"loss": np.asarray(r.train_loss)}
for i, (W, b) in enumerate(r.params):
    out[f"W{i}"] = W
    out[f"b{i}"] = b
np.savez(sys.argv[2], **out)
'''


def run(libdir, workload, path):
    env = dict(os.environ, GP_LIBDIR=os.path.abspath(libdir))
    subprocess.run([sys.executable, "-c", CHILD, workload, path], env=env, check=True)
    return np.load(path)


def main():
    a, b = sys.argv[1], sys.argv[2]
    workload = sys.argv[4] if len(sys.argv) > 4 and sys.argv[3] == "--workload" else "er"
    ra = run(a, workload, "/tmp/ab_a.npz")
    rb = run(b, workload, "/tmp/ab_b.npz")
    same = all(np.array_equal(ra[k].view(np.uint32), rb[k].view(np.uint32)) for k in ra.files)
    worst = max((float(np.max(np.abs(ra[k] - rb[k]))) for k in ra.files if ra[k].size), default=0.0)
    print(f"{workload}: bitwise_equal={same} max_abs_diff={worst:.3g} loss_a={ra['loss'][-1]:.7f} loss_b={rb['loss'][-1]:.7f}")
    sys.exit(0 if same else 1)


if __name__ == "__main__":
    main()
