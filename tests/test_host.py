"""CPU tests of the product's host layer (libgnnsim_b200.so, gs_* C-ABI): CSR build,
normalisation, dataset I/O, chunking, schedule and initialisation must be BIT-EXACT with
the reference (golden fixtures) and with the C oracle."""
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def ds(gp):
    return gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)


def test_csr_normalisation_features_bitexact(gp, ds):
    g = golden("graph_er500")
    off, nb, dg = ds.graph()
    assert np.array_equal(off, g["csr_offsets"]) and np.array_equal(nb, g["csr_neighbors"])
    assert np.array_equal(dg, g["degrees"])
    o, c, v = ds.normalize_adjacency()
    assert np.array_equal(o, g["norm_offsets"]) and np.array_equal(c, g["norm_cols"])
    assert np.array_equal(bits(v), bits(g["norm_vals"]))
    x, lab, sp = ds.arrays()
    assert np.array_equal(bits(x), bits(g["features"]))
    assert np.array_equal(lab, g["labels"]) and np.array_equal(sp, g["split"])


@pytest.mark.parametrize("K", [1, 4, 7])
def test_make_chunks_and_partition_bitexact(gp, ds, K):
    ref = golden(f"chunks_er500_k{K}")
    assert np.array_equal(gp.make_chunks(ds, K, 5), ref["chunk_of"])
    a, cut, bt = gp.partition_vertices(ds, K, 5)
    assert np.array_equal(a, ref["assignment"])
    assert cut == int(ref["edge_cut"][0]) and bt == int(ref["boundary_sizes"].sum())


def test_shuffle_order_and_stage_assignment_bitexact(gp):
    s = golden("shuffle_k8")
    assert np.array_equal(np.concatenate([gp.shuffle_chunk_order(8, t, 3) for t in range(1, 21)]), s["orders"])
    rows, i = s["stage_ranges"].reshape(-1, 4), 0
    for L in (1, 3, 8, 16, 64):
        for S in range(1, min(L, 8) + 1):
            for lo, hi in gp.make_stage_assignment(L, S):
                assert tuple(rows[i]) == (L, S, lo, hi)
                i += 1


@pytest.mark.parametrize("name,kind,layers", [("forward_gcn", 0, 3), ("forward_gcnii", 2, 5)])
def test_init_params_bitexact(gp, name, kind, layers):
    ref = golden(name)
    ps = gp.init_params(gp.ModelConfig(kind=kind, layers=layers, hidden=16), 16, 5, 7)
    for l, (W, b) in enumerate(ps):
        assert np.array_equal(bits(W), bits(ref[f"init_W{l}"]))
        assert np.array_equal(b, ref[f"init_b{l}"])


def test_layer_specs_gcnii_beta_schedule(gp):
    """beta_j = ln(lambda / j + 1) (nn.cpp:52-57, test_nn.cpp:432-452)."""
    specs = gp.build_layer_specs(gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=10, hidden=32), 7, 3)
    assert [s.kind for s in specs] == [0] + [3] * 8 + [0]
    for j, s in enumerate(specs[1:-1], start=1):
        assert s.beta == np.log(0.5 / j + 1.0) and s.alpha == 0.1
    assert specs[0].relu and not specs[-1].relu and (specs[0].in_dim, specs[-1].out_dim) == (7, 3)


@pytest.mark.parametrize("seed,n,p,K", [(1, 300, 0.03, 5), (2, 800, 0.008, 9), (3, 60, 0.2, 60)])
def test_host_matches_c_oracle_on_random_graphs(gp, seed, n, p, K):
    d = gp.Dataset.synthetic_er(n, p, seed, 6, 3, seed)
    o = O.OracleData.synthetic_er(n, p, seed, 6, 3, seed)
    for a, b in zip(d.graph(), o.graph()):
        assert np.array_equal(a, b)
    assert np.array_equal(gp.make_chunks(d, K, seed), o.partition(K, seed))
    assert np.array_equal(gp.shuffle_chunk_order(K, seed, 11), O.shuffle(K, seed, 11))


def test_build_graph_dedupes_and_drops_self_loops(gp):
    """test_graph.cpp:12-20."""
    d = gp.Dataset.from_edges(3, np.array([(0, 1), (1, 0), (0, 1), (2, 2), (1, 2)], np.uint32),
                              np.zeros((3, 1), np.float32), np.zeros(3, np.uint32), 1, np.ones(3, np.uint8))
    off, nb, deg = d.graph()
    assert d.num_edges == 2 and deg[1] == 2 and list(nb[off[1]:off[2]]) == [0, 2]


def test_er_extremes(gp):
    """test_graph.cpp:37-43."""
    assert gp.Dataset.synthetic_er(100, 0.0, 7, 1, 1, 1).num_edges == 0
    assert gp.Dataset.synthetic_er(100, 1.0, 7, 1, 1, 1).num_edges == 4950


def test_dataset_round_trip(gp, ds, tmp_path):
    """dataset.cpp:64-145 (test_dataset.cpp:81-90): save -> load -> save is byte-identical."""
    a, b = tmp_path / "a", tmp_path / "b"
    ds.save(str(a))
    d2 = gp.Dataset.load(str(a))
    d2.save(str(b))
    for f in ("meta.json", "graph.txt", "features.f32", "labels.u32", "masks.u8"):
        assert (a / f).read_bytes() == (b / f).read_bytes(), f
    for x, y in zip(ds.graph(), d2.graph()):
        assert np.array_equal(x, y)
    assert (a / "meta.json").read_text().startswith('{\n  "num_classes": 5,')


def test_load_reference_written_dataset(gp, tmp_path):
    from oracle.blob import have_ref
    import subprocess
    if not have_ref():
        pytest.skip("reference build absent")
    from oracle.blob import REF_DRIVER
    d = tmp_path / "sbm"
    subprocess.run([REF_DRIVER, "save", "spec=sbm:3:30:0.3:0.01:4", f"dir={d}"], check=True)
    ds = gp.Dataset.load(str(d))
    assert ds.num_vertices == 90 and ds.num_classes == 3 and ds.num_features == 3


def test_load_errors(gp, tmp_path):
    with pytest.raises(gp.GnnsimError):
        gp.Dataset.load(str(tmp_path / "missing"))


def test_invalid_arguments(gp, ds):
    with pytest.raises(gp.InvalidArgument):
        gp.make_chunks(ds, 501, 1)
    with pytest.raises(gp.InvalidArgument):
        gp.make_stage_assignment(4, 5)
    with pytest.raises(gp.InvalidArgument):
        gp.build_layer_specs(gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=2), 4, 2)


def test_powerlaw_dataset_chunk_plan_matches_reference():
    """make_chunks on the committed power-law fixture (load_dataset of a save_dataset directory)
    equals the reference's plan stored with its training goldens."""
    import paper_2308_10087_b200 as gp
    here = os.path.dirname(os.path.abspath(__file__))
    ds = gp.Dataset.load(os.path.join(here, "golden", "powerlaw_2k"))
    for name, K, seed in (("train_gcnii_powerlaw_hyb_s2g2", 4, 3), ("train_gcn_powerlaw_s2k8", 8, 4)):
        ref = np.load(os.path.join(here, "golden", name + ".npz"))
        assert np.array_equal(gp.make_chunks(ds, K, seed), ref["chunk_of"]), name


def test_dataset_binary_csr_cache_round_trip(tmp_path):
    """save_dataset writes graph.csr next to graph.txt (f2: binary CSR cache); load_dataset uses it
    only while graph.txt is unchanged, and both paths give the same graph."""
    import paper_2308_10087_b200 as gp
    ds = gp.Dataset.synthetic_er(3000, 0.004, 9, 8, 3, 2)
    d = tmp_path / "ds"
    ds.save(str(d))
    assert (d / "graph.csr").exists() and (d / "graph.txt").exists()
    a = gp.Dataset.load(str(d))
    for x, y in zip(a.graph(), ds.graph()):
        assert np.array_equal(x, y)
    # a stale cache is ignored: rewrite graph.txt with one edge removed
    lines = (d / "graph.txt").read_text().splitlines()
    n, m = (int(t) for t in lines[0].split())
    (d / "graph.txt").write_text(f"{n} {m - 1}\n" + "\n".join(lines[2:]) + "\n")
    meta = (d / "meta.json").read_text().replace(f'"num_edges": {m}', f'"num_edges": {m - 1}')
    (d / "meta.json").write_text(meta)
    b = gp.Dataset.load(str(d))
    assert b.num_edges == m - 1
    # the reference reads the same directory (graph.csr is an extra file it ignores)
    (d / "graph.csr").unlink()
    c = gp.Dataset.load(str(d))
    for x, y in zip(b.graph(), c.graph()):
        assert np.array_equal(x, y)


def test_assignment_files_match_reference_bytes(gp, tmp_path):
    """save_assignment / load_assignment (partition.cpp:250-269): chunks.txt and parts.txt byte-equal
    to the reference writer's, and loading either gives back the plan."""
    import os

    import numpy as np
    ref = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "assign_er500_k4.npz")))
    ds = gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)
    co = gp.make_chunks(ds, 4, 5)
    part, _, _ = gp.partition_vertices(ds, 4, 5)
    for name, arr in (("chunks.txt", co), ("parts.txt", part)):
        path = str(tmp_path / name)
        gp.save_assignment(path, 4, arr)
        assert open(path).read() == str(ref["file_" + name.replace(".", "_")]), name
        parts, back = gp.load_assignment(path)
        assert parts == 4 and np.array_equal(back, arr)
    ref_path = tmp_path / "ref_chunks.txt"
    ref_path.write_text(str(ref["file_chunks_txt"]))
    parts, back = gp.load_assignment(str(ref_path))
    assert parts == 4 and np.array_equal(back, ref["chunk_of"])
    bad = tmp_path / "bad.txt"
    bad.write_text("x\n")
    with pytest.raises(gp.GnnsimError):
        gp.load_assignment(str(bad))


def test_train_tool_partition_files_roundtrip(gp):
    """tools/gnnpipe_train.py --parts-file: the boundary total computed from a loaded parts.txt equals
    partition_vertices' own (partition.cpp:28-50)."""
    import numpy as np
    ds = gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)
    part, _, bt = gp.partition_vertices(ds, 3, 4)
    off, cols, _ = ds.normalize_adjacency(True)
    rows = np.repeat(np.arange(ds.num_vertices, dtype=np.int64), np.diff(off).astype(np.int64))
    cross = part[rows] != part[cols]
    assert int(np.unique(rows[cross] * 3 + part[cols[cross]]).size) == bt
