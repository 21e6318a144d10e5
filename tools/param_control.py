"""Engine-vs-engine control for long training goldens: how far two fp32 summation orders of the
engine drift apart (per-layer median relative parameter difference), next to engine vs reference."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_10087_b200 as gp  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def stats(params, ref):
    med, mx = [], []
    for l, (W, _) in enumerate(params):
        rW = ref[l].astype(np.float64)
        d = np.abs(W - rW) / np.maximum(np.abs(rW), 1e-3)
        med.append(float(np.median(d)))
        mx.append(float(np.abs(W - rW).max()))
    return med, mx


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg1_arxiv_gcn16_s2k8_20ep"
    g = dict(np.load(os.path.join(GOLD, name + ".npz")))
    ds = gp.Dataset.synthetic_er(169343, 2332486 / (169343 * 169342), 1, 128, 40, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCN, layers=16, hidden=128)
    co = gp.make_chunks(ds, 8, 1)
    runs = {}
    for tag, env in (("default", {}), ("simt_pgrad", {"GP_PGRAD": "simt"}), ("cuda_core", {"GP_TC_XFORM": "0"}),
                     ("cuda_core_simt", {"GP_TC_XFORM": "0", "GP_PGRAD": "simt"})):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        r = gp.train_pipeline(ds, co, 2, gp.TrainOptions(model=model, epochs=20, seed=1))
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v
        runs[tag] = [W for W, _ in r.params]
        med, mx = stats(r.params, [g[f"W{l}"] for l in range(16)])
        print(f"{tag:15s} vs reference: median rel per layer max {max(med):.2e} "
              f"{[f'{m:.1e}' for m in med]} absmax {max(mx):.2e}")
    base = runs["default"]
    for tag in ("simt_pgrad", "cuda_core", "cuda_core_simt"):
        med, mx = stats([(W, None) for W in runs[tag]], base)
        print(f"{tag:15s} vs default:   median rel per layer max {max(med):.2e} "
              f"{[f'{m:.1e}' for m in med]} absmax {max(mx):.2e}")


if __name__ == "__main__":
    main()
