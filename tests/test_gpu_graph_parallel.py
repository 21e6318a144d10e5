"""train_graph_parallel (engines_impl.hpp:320-479) on the GPU engine: per-layer halo
exchange + rank-ordered weight-gradient fold, against the reference's own outputs."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name,kind,L,P,ps,seed", [("train_gcn_graph_p3", 0, 3, 3, 5, 53),
                                                   ("train_gcnii_graph_p2", 2, 5, 2, 6, 54)])
def test_train_graph_parallel_matches_reference(gp, name, kind, L, P, ps, seed):
    if gp.device_count() == 0:
        pytest.fail("no CUDA device visible")
    ref = dict(np.load(os.path.join(GOLD, name + ".npz")))
    ds = gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)
    part, _, _ = gp.partition_vertices(ds, P, ps)
    opt = gp.TrainOptions(model=gp.ModelConfig(kind=kind, layers=L, hidden=16), epochs=6, seed=seed)
    res = gp.train_graph_parallel(ds, part, opt)
    met = ref["metrics"].reshape(6, 5)
    assert np.max(np.abs(res.train_loss - met[:, 1]) / np.abs(met[:, 1])) < 1e-4
    assert np.array_equal(res.comm.astype(np.uint64), ref["comm"].reshape(6, 3))
    for l, (W, b) in enumerate(res.params):
        rW = ref[f"W{l}"]
        assert float(np.max(np.abs(W - rW) / np.maximum(np.abs(rW), 1e-3))) < 2e-3
