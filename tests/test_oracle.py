"""Pins the C restatement oracle (oracle/gnnsim_oracle.c) to the reference.

1. against the golden fixtures generated from the reference build (tests/golden/);
2. against the reference's own in-code known answers (proj/tests/test_graph.cpp,
   test_partition.cpp, test_engines.cpp);
3. against the live reference binary on extra scenarios, when oracle/_ref/ref_driver exists.
The bar is bit-exactness everywhere: same libstdc++ <random> algorithms, same glibc libm,
same scalar float operation order.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle.blob import have_ref, run_ref

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def er500():
    return O.OracleData.synthetic_er(500, 0.02, 3, 16, 5, 9)


def test_graph_and_features_match_golden(er500):
    g = golden("graph_er500")
    off, nb, dg = er500.graph()
    assert np.array_equal(off, g["csr_offsets"]) and np.array_equal(nb, g["csr_neighbors"])
    assert np.array_equal(dg, g["degrees"]) and er500.m == int(g["num_edges"][0])
    o, c, v = er500.normalize()
    assert np.array_equal(o, g["norm_offsets"]) and np.array_equal(c, g["norm_cols"])
    assert np.array_equal(bits(v), bits(g["norm_vals"]))
    x, lab, sp = er500.arrays()
    assert np.array_equal(bits(x), bits(g["features"]))
    assert np.array_equal(lab, g["labels"]) and np.array_equal(sp, g["split"])


@pytest.mark.parametrize("K", [1, 4, 7])
def test_chunks_match_golden(er500, K):
    assert np.array_equal(er500.partition(K, 5), golden(f"chunks_er500_k{K}")["chunk_of"])


def test_sbm_chunks_recover_blocks_like_reference():
    """test_partition.cpp:128-139 + golden chunk_of on the reference's own SBM graph."""
    g = golden("graph_sbm4x100")
    off, nb = g["csr_offsets"], g["csr_neighbors"]
    n = len(off) - 1
    edges = [(v, u) for v in range(n) for u in nb[off[v]:off[v + 1]] if v < u]
    d = O.OracleData.from_edges(n, np.array(edges, np.uint32), g["features"], g["labels"], 4, g["split"])
    co = d.partition(4, 31)
    assert np.array_equal(co, golden("chunks_sbm4x100_k4")["chunk_of"])
    majority = sorted(int(np.bincount(np.arange(n)[co == k] // 100, minlength=4).argmax()) for k in range(4))
    assert majority == [0, 1, 2, 3]


def test_shuffle_and_stage_ranges_match_golden():
    s = golden("shuffle_k8")
    assert np.array_equal(np.concatenate([O.shuffle(8, t, 3) for t in range(1, 21)]), s["orders"])
    rows, i = s["stage_ranges"].reshape(-1, 4), 0
    for L in (1, 3, 8, 16, 64):
        for S in range(1, min(L, 8) + 1):
            for lo, hi in O.stage_ranges(L, S):
                assert tuple(rows[i]) == (L, S, lo, hi)
                i += 1


@pytest.mark.parametrize("name,kind,layers", [("forward_gcn", 0, 3), ("forward_gcnii", 2, 5)])
def test_init_params_match_golden(name, kind, layers):
    ref = golden(name)
    count = sum(ref[f"init_W{l}"].size + ref[f"init_b{l}"].size for l in range(layers))
    flat = O.init_params(kind, layers, 16, 16, 5, 7, count)
    want = np.concatenate([np.concatenate([ref[f"init_W{l}"].ravel(), ref[f"init_b{l}"]]) for l in range(layers)])
    assert np.array_equal(bits(flat), bits(want))


def _params(ref, L):
    return np.concatenate([np.concatenate([ref[f"W{l}"].ravel(), ref[f"b{l}"]]) for l in range(L)])


TRAIN = [
    # golden name, ds, model, L, H, S, K, chunk seed, epochs, seed, extra
    ("train_gcn_s1k1", "er500", 0, 4, 16, 1, 1, 1, 10, 42, {}),
    ("train_gcn_s2k4", "er500", 0, 4, 16, 2, 4, 3, 10, 42, dict(fix_alpha=3)),
    ("train_gcnii_s2k4", "er500", 2, 6, 16, 2, 4, 3, 10, 43, dict(fix_alpha=3)),
    ("train_gcnii_s1k4_sync", "er500", 2, 6, 16, 1, 4, 3, 10, 44, dict(sync=True)),
    ("train_gcn_s3k6_w40", "er300w", 0, 6, 24, 3, 6, 1, 8, 45, dict(fix_alpha=2)),
]


@pytest.mark.parametrize("case", TRAIN, ids=[c[0] for c in TRAIN])
def test_training_bitexact_with_reference_golden(er500, case):
    name, dsn, model, L, H, S, K, cs, ep, seed, kw = case
    ref = golden(name)
    d = er500 if dsn == "er500" else O.OracleData.synthetic_er(300, 0.03, 11, 40, 7, 2)
    co = np.zeros(d.n, np.uint32) if K == 1 else d.partition(K, cs)
    want = _params(ref, L)
    met, comm, params, _ = d.train(co, K, S, model, L, H, seed, ep, num_params=want.size, **kw)
    assert np.array_equal(met, ref["metrics"].reshape(ep, 5))
    assert np.array_equal(bits(params), bits(want))
    assert np.array_equal(comm, ref["comm"].reshape(ep, 3)[:, 1])


def test_reference_kats_normalisation():
    """test_graph.cpp:62-88: isolated vertex -> 1, K2 -> four 0.5, star -> 1/4 and 1/sqrt(8)."""
    def norm(n, edges):
        d = O.OracleData.from_edges(n, np.array(edges, np.uint32), np.zeros((n, 1), np.float32),
                                    np.zeros(n, np.uint32), 1, np.ones(n, np.uint8))
        return d.normalize()
    off, col, val = norm(3, [(0, 1)])
    assert off[3] - off[2] == 1 and col[off[2]] == 2 and val[off[2]] == 1.0
    _, _, val = norm(2, [(0, 1)])
    assert list(val) == [0.5] * 4
    off, col, val = norm(4, [(0, 1), (0, 2), (0, 3)])
    for i in range(off[0], off[1]):
        want = 0.25 if col[i] == 0 else 1 / np.sqrt(8.0)
        assert abs(val[i] - want) < 1e-7


def test_reference_kat_two_triangles_zero_cut():
    """test_partition.cpp:13-21."""
    d = O.OracleData.from_edges(6, np.array([(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)], np.uint32),
                                np.zeros((6, 1), np.float32), np.zeros(6, np.uint32), 1, np.ones(6, np.uint8))
    p = d.partition(2, 9)
    off, nb, _ = d.graph()
    assert all(p[v] == p[u] for v in range(6) for u in nb[off[v]:off[v + 1]])
    assert sorted(np.bincount(p)) == [3, 3]


def test_dropout_mask_rate_and_determinism():
    a = O.dropmask(0.5, 7, 3, 2, 1000, 64)
    b = O.dropmask(0.5, 7, 3, 2, 1000, 64)
    c = O.dropmask(0.5, 7, 4, 2, 1000, 64)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    ones = sum(bin(int(w)).count("1") for w in a)
    assert abs(ones / 64000 - 0.5) < 0.02


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref/ref_driver not built")
@pytest.mark.parametrize("kw", [
    dict(model="gcnii", layers=7, hidden=12, S=3, K=5, chunk_seed=4, epochs=6, seed=3, fix_alpha=2, hist=1),
    dict(model="gcn", layers=5, hidden=10, S=2, K=3, chunk_seed=2, epochs=5, seed=9, optimizer="sgd", lr=0.05),
    dict(model="gcnii", layers=4, hidden=8, S=4, K=8, chunk_seed=5, epochs=4, seed=2, shuffle=0, dropout=0.0),
], ids=["hist", "sgd", "noshuffle_nodropout"])
def test_training_bitexact_with_live_reference(tmp_path, kw):
    spec = "er:400:0.025:6:12:4:8"
    ref = run_ref("train", str(tmp_path / "t.blob"), spec=spec, **kw)
    d = O.OracleData.synthetic_er(400, 0.025, 6, 12, 4, 8)
    co = d.partition(kw["K"], kw["chunk_seed"])
    assert np.array_equal(co, ref["chunk_of"])
    L = kw["layers"]
    want = _params(ref, L)
    met, comm, params, _ = d.train(co, kw["K"], kw["S"], 2 if kw["model"] == "gcnii" else 0, L, kw["hidden"],
                                   kw["seed"], kw["epochs"], dropout=kw.get("dropout", 0.5),
                                   shuffle=bool(kw.get("shuffle", 1)), fix_alpha=kw.get("fix_alpha", 10),
                                   hist=bool(kw.get("hist", 0)), sgd=kw.get("optimizer") == "sgd",
                                   lr=kw.get("lr", 1e-3), num_params=want.size)
    assert np.array_equal(met, ref["metrics"].reshape(kw["epochs"], 5))
    assert np.array_equal(bits(params), bits(want))
