"""Per-layer accuracy of the row transforms against an fp64 evaluation of the same inputs.

One GCNII epoch (stage = whole model, K = 1) with the tcgen05 transforms (GP_TC_XFORM=1, 3xTF32)
and with the CUDA-core transforms (GP_TC_XFORM=0, the reference's sequential fp32 order). For each
Gcn2Conv layer the forward output h = relu(pre . W'), W' = beta W + (1 - beta) I (nn.hpp:183-196),
and the backward gather row bg = (1 - alpha) dz . W'^T (nn.hpp:202-218) are recomputed in fp64
from the run's own pre / dz, so each number is the error of that transform alone. Error = |x - x64| / max_row|x64|.

    python tools/xform_accuracy.py [N] [avg_degree] [layers]      (on the GPU box)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_10087_b200 as gp  # noqa: E402


def err(x, ref):
    scale = np.maximum(np.abs(ref).max(axis=1, keepdims=True), 1e-30)
    e = (np.abs(x.astype(np.float64) - ref) / scale).ravel()
    return np.median(e), np.quantile(e, 0.999), e.max()


def run(mode, ds, model, F, C):
    os.environ["GP_TC_XFORM"] = mode
    os.environ["GP_LEAN"] = "0"
    specs = gp.build_layer_specs(model, F, C)
    params = gp.init_params(model, F, C, 1)
    N = ds.num_vertices
    eng = gp.StageEngine(num_vertices=N, num_chunks=1, specs=specs, stage=0, num_stages=1,
                         layer_range=(0, len(specs)), hidden=model.hidden, num_classes=C, dropout=0.5, seed=1)
    off, cols, vals = ds.normalize_adjacency(True)
    eng.upload_graph(off, cols, vals, np.zeros(N, np.uint32))
    x, lab, sp = ds.arrays()
    eng.upload_features(x)
    eng.upload_labels(lab, sp)
    for l, (W, b) in enumerate(params):
        eng.set_params(l, W, b)
    eng.run_epoch(1, [0])
    out = []
    for l, s in enumerate(specs):
        if s.kind != gp.LayerKind.GCN2CONV:
            continue
        W = params[l][0].astype(np.float64)
        Wp = s.beta * W + (1.0 - s.beta) * np.eye(W.shape[0])
        pre = eng.download("pre", l).astype(np.float64)
        h = eng.download("h", l)
        h64 = pre @ Wp
        if s.relu:
            h64 = np.maximum(h64, 0.0)
        dz = eng.download("dz", l).astype(np.float64)
        bg = eng.download("dagg", l)  # the backward gather table: (1 - alpha) dagg for Gcn2Conv
        out.append((l, err(h, h64), err(bg, (1.0 - s.alpha) * (dz @ Wp.T))))
    eng.close()
    return out


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
    deg = float(sys.argv[2]) if len(sys.argv) > 2 else 50.0
    L = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    F, C, H = 100, 16, 100
    ds = gp.Dataset.synthetic_er(N, deg / (N - 1), 1, F, C, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=L, hidden=H)
    res = {m: run(m, ds, model, F, C) for m in ("1", "0")}
    print(f"N={N} avg_degree={deg} layers={L}: error / max_row|x64| (median, 99.9 %, max)")
    for (l, fh, bd), (_, fh0, bd0) in zip(res["1"], res["0"]):
        print(f"layer {l:2d} fwd h    tcgen05 {fh[0]:.1e} {fh[1]:.1e} {fh[2]:.1e} | cuda-core {fh0[0]:.1e} {fh0[1]:.1e} "
              f"{fh0[2]:.1e}")
        print(f"         bwd bg   tcgen05 {bd[0]:.1e} {bd[1]:.1e} {bd[2]:.1e} | cuda-core {bd0[0]:.1e} {bd0[1]:.1e} "
              f"{bd0[2]:.1e}")


if __name__ == "__main__":
    main()
