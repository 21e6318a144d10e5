"""GPU parity tests: the sm_100a engine (through the C-ABI) against the reference.

Ground truth, in order of preference:
  * golden fixtures produced by the unmodified reference (tests/golden/*.npz, make_golden.py);
  * the reference binary itself run live (oracle/_ref/ref_driver), when it was built.

Bars:
  * forward activations at epoch 1 (same parameters): BIT-EXACT — the kernels keep the
    reference's scalar operation order (ascending neighbours, mul then add, no FMA);
  * anything downstream of the softmax (expf/logf differ from glibc by <= 2 ulp) and the
    parameter gradients (split-K reduction order): relative 1e-4 on activations/gradients,
    loss-curve agreement rel 1e-4 over the run, parameters rel 2e-3 max / 1e-4 median;
  * communication ledger: exact.
"""
import os

import numpy as np
import pytest

from oracle.blob import have_ref, run_ref

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ER500 = (500, 0.02, 3, 16, 5, 9)


def golden(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


@pytest.fixture(scope="module", autouse=True)
def need_gpu(gp):
    if gp.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


def er500(gp):
    return gp.Dataset.synthetic_er(*ER500)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a, np.float32).view(np.uint32),
                          np.ascontiguousarray(b, np.float32).view(np.uint32))


def single_stage(gp, ds, model, seed, K=1, chunk_of=None, **kw):
    specs = gp.build_layer_specs(model, ds.num_features, ds.num_classes)
    L = len(specs)
    eng = gp.StageEngine(num_vertices=ds.num_vertices, num_chunks=K, specs=specs, stage=0, num_stages=1,
                         layer_range=(0, L), hidden=model.hidden, num_classes=ds.num_classes,
                         dropout=model.dropout, seed=seed, **kw)
    off, cols, vals = ds.normalize_adjacency(model.self_loops)
    co = np.zeros(ds.num_vertices, np.uint32) if chunk_of is None else chunk_of
    eng.upload_graph(off, cols, vals, co)
    x, lab, sp = ds.arrays()
    eng.upload_features(x)
    eng.upload_labels(lab, sp)
    for l, (W, b) in enumerate(gp.init_params(model, ds.num_features, ds.num_classes, seed)):
        eng.set_params(l, W, b)
    return eng, specs


@pytest.mark.parametrize("name,kind,layers", [("forward_gcn", 0, 3), ("forward_gcnii", 2, 5), ("forward_sage", 1, 3)])
def test_epoch1_forward_bitexact_and_backward_close(gp, name, kind, layers, monkeypatch):
    monkeypatch.setenv("GP_LEAN", "0")  # keep h apart from dz so the activations can be read back
    monkeypatch.setenv("GP_TC_XFORM", "0")  # the bit-exact CUDA-core transforms
    ref = golden(name)
    ds = er500(gp)
    model = gp.ModelConfig(kind=kind, layers=layers, hidden=16)
    eng, specs = single_stage(gp, ds, model, seed=7)
    st = eng.run_epoch(1, [0])
    for l in range(layers):
        assert bits_equal(eng.download("h", l), ref[f"h{l}"]), f"h{l} not bit-exact"
        assert bits_equal(eng.download("pre", l), ref[f"pre{l}"]), f"pre{l} not bit-exact"
    ntrain = int((ds.arrays()[2] == 1).sum())
    assert abs(st.loss_sum / ntrain - float(ref["loss"][0])) <= 1e-6 * abs(float(ref["loss"][0]))
    for l in range(layers):
        assert rel(eng.download("dz", l), ref[f"dz{l}"]) < 1e-4, f"dz{l}"
    for l in range(1, layers):
        got = eng.download("dagg", l)
        want = ref[f"dagg{l}"]
        if specs[l].kind == gp.LayerKind.GCN2CONV:  # engine stores (1-a)*dagg, rounded like nn.hpp:251
            want = np.float32(1.0 - np.float32(specs[l].alpha)) * want
        assert rel(got, want) < 1e-4, f"dagg{l}"
    if kind == 2:
        # dh0 accumulates a*dagg over the Gcn2Conv layers (nn.hpp:216)
        assert rel(eng.download("dh0"), ref["dh0"]) < 1e-4


@pytest.mark.parametrize("mode", ["tc", "simt"])
@pytest.mark.parametrize("name,kind,layers", [("forward_gcn", 0, 3), ("forward_gcnii", 2, 5), ("forward_sage", 1, 3)])
def test_param_grads_match_reference(gp, name, kind, layers, mode, monkeypatch):
    """param_grads_for_rows (nn.hpp:269-293): tcgen05 3xTF32 (default) and CUDA-core paths."""
    monkeypatch.setenv("GP_PGRAD", mode)
    ref = golden(name)
    ds = er500(gp)
    model = gp.ModelConfig(kind=kind, layers=layers, hidden=16)
    eng, specs = single_stage(gp, ds, model, seed=7)
    eng.run_epoch(1, [0])
    for l in range(layers):
        gW, gb = eng.get_grads(l)
        assert rel(gW, ref[f"gW{l}"]) < 1e-4, (mode, l, rel(gW, ref[f"gW{l}"]))
        if gb.size:
            assert rel(gb, ref[f"gb{l}"]) < 1e-4, (mode, l)


def test_param_grads_wide_layer_tc(gp, monkeypatch):
    """tcgen05 path with k_in = 300 (three M tiles, last partial) and N = 40 (padded to 48)."""
    monkeypatch.setenv("GP_PGRAD", "tc")
    ds = gp.Dataset.synthetic_er(2000, 0.004, 4, 300, 40, 6)
    model = gp.ModelConfig(kind=2, layers=3, hidden=40)
    eng, specs = single_stage(gp, ds, model, seed=3)
    eng.run_epoch(1, [0])
    pre = eng.download("pre", 0).astype(np.float64)
    dz = eng.download("dz", 0).astype(np.float64)
    gW, gb = eng.get_grads(0)
    assert rel(gW, pre.T @ dz) < 1e-5
    assert rel(gb, dz.sum(0)) < 1e-5


def test_params_after_one_adam_step(gp):
    ref = golden("forward_gcnii")
    ds = er500(gp)
    model = gp.ModelConfig(kind=2, layers=5, hidden=16)
    eng, specs = single_stage(gp, ds, model, seed=7)
    eng.run_epoch(1, [0])
    init = gp.init_params(model, ds.num_features, ds.num_classes, 7)
    for l, s in enumerate(specs):
        W, b = eng.get_params(l)
        g = ref[f"gW{l}"].astype(np.float64)
        # first Adam step: p -= lr * g / (|g| + eps) (bias-corrected moments)
        want = init[l][0].astype(np.float64) - 1e-3 * g / (np.abs(g) + 1e-8)
        assert np.max(np.abs(W - want)) < 2e-6, f"W{l}"


def _train_compare(gp, gname, ds, model, S, K, chunk_seed, epochs, seed, loss_tol=1e-4, acc_tol=None,
                   param_abs_tol=None, **stal):
    ref = golden(gname)
    chunk_of = np.zeros(ds.num_vertices, np.uint32) if K == 1 else gp.make_chunks(ds, K, chunk_seed)
    if K > 1 and ref["chunk_of"].size:
        assert np.array_equal(chunk_of, ref["chunk_of"]), "chunk plan not bit-exact"
    opt = gp.TrainOptions(model=model, epochs=epochs, seed=seed, **stal)
    res = gp.train_pipeline(ds, chunk_of, S, opt)
    met = ref["metrics"].reshape(epochs, 5)
    assert np.array_equal(res.metrics[:, 0], met[:, 0])
    assert np.max(np.abs(res.train_loss - met[:, 1]) / np.abs(met[:, 1])) < loss_tol, (res.train_loss, met[:, 1])
    # accuracies: allow a couple of argmax flips on near-ties
    n = ds.num_vertices
    assert np.max(np.abs(res.metrics[:, 2:5] - met[:, 2:5])) <= (acc_tol if acc_tol else 3.0 / (0.2 * n))
    comm = ref["comm"].reshape(epochs, 3)
    assert np.array_equal(res.comm.astype(np.uint64), comm), "ledger bytes differ"
    worst, med, absmax = 0.0, [], 0.0
    for l, (W, b) in enumerate(res.params):
        rW = ref[f"W{l}"]
        absmax = max(absmax, float(np.abs(W.astype(np.float64) - rW).max()))
        d = np.abs(W.astype(np.float64) - rW) / np.maximum(np.abs(rW), 1e-3)
        worst = max(worst, float(d.max()))
        med.append(float(np.median(d)))
    if param_abs_tol is None:
        assert worst < 2e-3 and max(med) < 1e-4, (worst, med)
    else:  # long / deep runs: bounded in units of Adam steps (see the caller)
        assert absmax <= param_abs_tol and max(med) < 1e-3, (absmax, med)
    return res


def test_train_gcn_full_graph_matches_sequential_oracle(gp):
    _train_compare(gp, "train_gcn_s1k1", er500(gp), gp.ModelConfig(kind=0, layers=4, hidden=16), 1, 1, 1, 10, 42)


def test_train_gcn_pipeline_stale_two_stages(gp):
    _train_compare(gp, "train_gcn_s2k4", er500(gp), gp.ModelConfig(kind=0, layers=4, hidden=16), 2, 4, 3, 10, 42,
                   fix_alpha=3)


@pytest.mark.parametrize("env", [{}, {"GP_SPLIT": "0"}, {"GP_WAVE": "1"}, {"GP_OCC5": "0"}, {"GP_MERGED_G": "0"},
                                 {"GP_LEAN": "0"}],
                         ids=["default", "fused", "one_stream", "occ4", "split_g", "swap_layout"])
def test_train_sage_pipeline_stale_two_stages(gp, env, monkeypatch):
    """GraphSAGE (SageConv: [own | mean] . W, nn.hpp:176-182, :234-243) over two stages, under every
    engine variant switch (SageConv layers always run split; the others follow GP_SPLIT)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _train_compare(gp, "train_sage_s2k4", er500(gp), gp.ModelConfig(kind=1, layers=4, hidden=16), 2, 4, 3, 10, 46,
                   fix_alpha=3)


def test_sage_wide_features_forward_bitexact(gp, monkeypatch):
    """SageConv layer 0 over F = 200 features (> 128): mean aggregate + own row through the wide
    path (k_spmm_pre, k_remask, k_dense_gemm with the gapped weights), bit-exact."""
    monkeypatch.setenv("GP_LEAN", "0")
    monkeypatch.setenv("GP_TC_XFORM", "0")
    ref = golden("forward_sage_wide")
    ds = gp.Dataset.synthetic_er(300, 0.03, 11, 200, 7, 2)
    model = gp.ModelConfig(kind=1, layers=3, hidden=16)
    eng, specs = single_stage(gp, ds, model, seed=7)
    st = eng.run_epoch(1, [0])
    for l in range(3):
        assert bits_equal(eng.download("h", l), ref[f"h{l}"]), f"h{l} not bit-exact"
        assert bits_equal(eng.download("pre", l), ref[f"pre{l}"]), f"pre{l} not bit-exact"
    ntrain = int((ds.arrays()[2] == 1).sum())
    assert abs(st.loss_sum / ntrain - float(ref["loss"][0])) <= 1e-6 * abs(float(ref["loss"][0]))
    for l in range(3):
        gW, gb = eng.get_grads(l)
        assert rel(gW, ref[f"gW{l}"]) < 1e-4, l


def test_train_sage_wide_features_two_stages(gp):
    _train_compare(gp, "train_sage_wide_s2k4", gp.Dataset.synthetic_er(300, 0.03, 11, 200, 7, 2),
                   gp.ModelConfig(kind=1, layers=3, hidden=16), 2, 4, 1, 6, 50, fix_alpha=2)


# (base env, variant env): the fused kernels (GP_SPLIT=0) run the CUDA-core GEMV, so they are
# compared with the CUDA-core split transforms (GP_TC_XFORM=0)
CC = {"GP_TC_XFORM": "0"}
VARIANTS = [(CC, {"GP_SPLIT": "0"}), ({}, {"GP_WAVE": "1"}), ({}, {"GP_OCC5": "0"}), ({}, {"GP_PGRAD": "simt"}),
            ({}, {"GP_MERGED_G": "0"}), (CC, {"GP_MERGED_G": "0", "GP_SPLIT": "0"}), ({}, {"GP_LEAN": "0"}),
            ({}, {"GP_LEAN": "0", "GP_MERGED_G": "0"}), (CC, {"GP_LEAN": "0", "GP_SPLIT": "0"}),
            (CC, {"GP_WAVE": "1"}), (CC, {"GP_LEAN": "0"}), ({}, {"GP_BWD_CSR": "0"}),
            (CC, {"GP_BWD_CSR": "0", "GP_SPLIT": "0"}), ({}, {"GP_REMASK_OVERLAP": "0"}),
            ({}, {"GP_REMASK_OVERLAP": "0", "GP_WAVE": "1"}), ({}, {"GP_XF_PAD": "0"}),
            ({}, {"GP_GRAPH_BUILD": "device"}), ({}, {"GP_FUSED_STEP": "0"})]
VARIANT_IDS = ["fused", "one_stream", "occ4", "simt_pgrad", "split_g", "split_g_fused", "swap_layout",
               "swap_layout_split_g", "swap_layout_fused", "cuda_core_one_stream", "cuda_core_swap_layout",
               "batch_filter", "batch_filter_fused", "remask_in_order", "remask_in_order_one_stream",
               "xf_dense_stride", "device_graph_build", "per_layer_step"]


@pytest.mark.parametrize("hist", [False, True], ids=["stale", "hist"])
@pytest.mark.parametrize("G", [1, 2], ids=["pipeline", "hybrid"])
@pytest.mark.parametrize("envs", VARIANTS, ids=VARIANT_IDS)
def test_engine_variants_match_default_bitwise(gp, envs, G, hist, monkeypatch):
    """The engine's switches change scheduling, kernel shapes and the stash layout (lean
    in-place dz / bg-in-G with snapshot copies vs separate buffers with pointer swaps), never
    arithmetic order (except the pgrad reduction): losses and parameters equal the default run
    bit for bit, in pipeline and hybrid runs, with and without historical gradients."""
    ds = er500(gp)
    model = gp.ModelConfig(kind=2, layers=6, hidden=16)
    co = gp.make_chunks(ds, 4, 3)
    part, _, _ = gp.partition_vertices(ds, 2, 2)

    def run():
        opt = gp.TrainOptions(model=model, epochs=4, seed=9, fix_alpha=2, historical_gradients=hist)
        if G == 1:
            return gp.train_pipeline(ds, co, 2, opt)
        return gp.train_hybrid(ds, part, co, 2, opt)

    base_env, env = envs
    for k, v in base_env.items():
        monkeypatch.setenv(k, v)
    base = run()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    res = run()
    if "GP_PGRAD" in env:  # different parameter-gradient summation order: tolerance
        np.testing.assert_allclose(res.train_loss, base.train_loss, rtol=1e-4)
        return
    np.testing.assert_array_equal(res.train_loss, base.train_loss)
    for (Wa, _), (Wb, _) in zip(res.params, base.params):
        assert np.array_equal(Wa.view(np.uint32), Wb.view(np.uint32))


def test_train_sage_historical_gradients(gp):
    _train_compare(gp, "train_sage_s1k4_hist", er500(gp), gp.ModelConfig(kind=1, layers=3, hidden=16), 1, 4, 3, 8, 47,
                   fix_alpha=2, historical_gradients=True)


@pytest.mark.parametrize("mix", ["0", "1"], ids=["folded_mix", "epilogue_mix"])
def test_train_gcnii_pipeline_stale_two_stages(gp, mix, monkeypatch):
    """GCNII over two stages, 10 epochs; with the identity mix folded into the tcgen05 operand
    (default) and applied in the transform epilogue (GP_TC_MIX=1)."""
    monkeypatch.setenv("GP_TC_MIX", mix)
    _train_compare(gp, "train_gcnii_s2k4", er500(gp), gp.ModelConfig(kind=2, layers=6, hidden=16), 2, 4, 3, 10, 43,
                   fix_alpha=3)


def test_train_gcnii_synchronous_mode(gp):
    _train_compare(gp, "train_gcnii_s1k4_sync", er500(gp), gp.ModelConfig(kind=2, layers=6, hidden=16), 1, 4, 3,
                   10, 44, synchronous_mode=True)


def test_train_gcn_three_stages_wide_features(gp):
    ds = gp.Dataset.synthetic_er(300, 0.03, 11, 40, 7, 2)
    _train_compare(gp, "train_gcn_s3k6_w40", ds, gp.ModelConfig(kind=0, layers=6, hidden=24), 3, 6, 1, 8, 45,
                   fix_alpha=2)


def test_pipeline_ledger_closed_form(gp):
    """comm_bytes_pipeline == 2(S-1) N H vecs 4 exactly (analytics.cpp:12-15, test_engines.cpp:193-211)."""
    ds = er500(gp)
    for kind, vecs in ((0, 1), (2, 2)):
        for S in (2, 4):
            model = gp.ModelConfig(kind=kind, layers=8, hidden=16)
            co = gp.make_chunks(ds, 4 * S, 12)
            res = gp.train_pipeline(ds, co, S, gp.TrainOptions(model=model, epochs=2, seed=50))
            want = 2 * (S - 1) * ds.num_vertices * 16 * 4 * vecs
            assert all(int(c[1]) == want for c in res.comm), (res.comm, want)
            assert all(int(c[0]) == 0 and int(c[2]) == 0 for c in res.comm)


@pytest.mark.parametrize("row_order", ["id", "degree"])
def test_stale_equals_exact_on_chunk_disconnected_graph(gp, row_order, monkeypatch):
    """test_engines.cpp:138-155: no cross-chunk edge -> stale pipeline == full-graph run.

    With GP_ROW_ORDER=id both runs reduce parameter gradients over rows in the same
    (id) order and must agree bit for bit, as in the reference. The default
    (chunk, degree) row order changes that reduction order between K=1 and K=2, so
    the runs then agree to rounding only."""
    monkeypatch.setenv("GP_ROW_ORDER", row_order)
    n = 80
    rng = np.random.default_rng(9)
    edges = [(u, v) for u in range(n) for v in range(u + 1, n) if u // 40 == v // 40 and rng.random() < 0.3]
    x = rng.standard_normal((n, 8)).astype(np.float32)
    lab = (np.arange(n) // 40).astype(np.uint32)
    sp = np.ones(n, np.uint8)
    ds = gp.Dataset.from_edges(n, np.array(edges, np.uint32), x, lab, 2, sp)
    model = gp.ModelConfig(kind=0, layers=4, hidden=8)
    opt = gp.TrainOptions(model=model, epochs=5, seed=46)
    seq = gp.train_sequential(ds, opt)
    pipe = gp.train_pipeline(ds, (np.arange(n) // 40).astype(np.uint32), 2, opt)
    for (a, _), (b, _) in zip(seq.params, pipe.params):
        if row_order == "id":
            assert bits_equal(a, b)
        else:
            assert rel(a, b) < 1e-5
    if row_order == "id":
        assert np.array_equal(seq.train_loss, pipe.train_loss)
    else:
        np.testing.assert_allclose(seq.train_loss, pipe.train_loss, rtol=1e-6)


def test_deterministic_reruns(gp):
    ds = er500(gp)
    model = gp.ModelConfig(kind=2, layers=6, hidden=16)
    co = gp.make_chunks(ds, 4, 3)
    a = gp.train_pipeline(ds, co, 2, gp.TrainOptions(model=model, epochs=3, seed=1))
    b = gp.train_pipeline(ds, co, 2, gp.TrainOptions(model=model, epochs=3, seed=1))
    assert np.array_equal(a.train_loss, b.train_loss)
    for (x, _), (y, _) in zip(a.params, b.params):
        assert bits_equal(x, y)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref/ref_driver not built")
def test_live_reference_gcnii_three_stages(gp, tmp_path):
    spec = "er:700:0.015:5:24:6:4"
    ds = gp.Dataset.synthetic_er(700, 0.015, 5, 24, 6, 4)
    kw = dict(model="gcnii", layers=9, hidden=32, S=3, K=6, chunk_seed=2, epochs=20, seed=8, fix_alpha=4)
    ref = run_ref("train", str(tmp_path / "t.blob"), spec=spec, **kw)
    co = gp.make_chunks(ds, 6, 2)
    assert np.array_equal(co, ref["chunk_of"])
    opt = gp.TrainOptions(model=gp.ModelConfig(kind=2, layers=9, hidden=32), epochs=20, seed=8, fix_alpha=4)
    res = gp.train_pipeline(ds, co, 3, opt)
    met = ref["metrics"].reshape(20, 5)
    assert np.max(np.abs(res.train_loss - met[:, 1]) / met[:, 1]) < 1e-4
    assert np.array_equal(res.comm.astype(np.uint64), ref["comm"].reshape(20, 3))


def test_invalid_arguments_raise(gp):
    ds = er500(gp)
    model = gp.ModelConfig(kind=0, layers=4, hidden=16)
    with pytest.raises(gp.InvalidArgument):
        gp.train_pipeline(ds, np.zeros(ds.num_vertices, np.uint32), 5, gp.TrainOptions(model=model))
    with pytest.raises(gp.InvalidArgument):
        gp.train_pipeline(ds, np.arange(ds.num_vertices, dtype=np.uint32) % 65, 1, gp.TrainOptions(model=model))
    # SageConv hidden widths above 128 are not supported by the row kernels
    with pytest.raises(gp.InvalidArgument, match="SageConv"):
        gp.train_pipeline(ds, np.zeros(ds.num_vertices, np.uint32), 1,
                          gp.TrainOptions(model=gp.ModelConfig(kind=1, layers=3, hidden=136)))


HYB = [
    # golden, model kind, L, H, S, G, K, chunk seed, part seed, epochs, seed, staleness kwargs
    ("train_gcn_hyb_s2g2", 0, 4, 16, 2, 2, 4, 3, 1, 8, 42, dict(fix_alpha=3)),
    ("train_gcnii_hyb_s2g2", 2, 6, 16, 2, 2, 4, 3, 2, 8, 43, dict(fix_alpha=3)),
    ("train_gcnii_hyb_s1g3_sync", 2, 5, 16, 1, 3, 3, 5, 3, 6, 44, dict(synchronous_mode=True)),
    ("train_gcn_hyb_s3g2_hist", 0, 6, 12, 3, 2, 6, 7, 4, 6, 45, dict(fix_alpha=2, historical_gradients=True)),
    ("train_sage_hyb_s2g2", 1, 4, 16, 2, 2, 4, 3, 1, 8, 48, dict(fix_alpha=3)),
    ("train_sage_hyb_s1g2_hist", 1, 3, 12, 1, 2, 4, 5, 2, 6, 49, dict(fix_alpha=2, historical_gradients=True)),
]


@pytest.mark.parametrize("case", HYB, ids=[c[0] for c in HYB])
def test_train_hybrid_matches_reference(gp, case):
    """train_hybrid (engines_impl.hpp:515-909) with G graph partitions per stage: halo
    exchange, rank-ordered weight-gradient fold; ledger exact for all three classes."""
    name, kind, L, H, S, G, K, cs, ps, ep, seed, kw = case
    ref = golden(name)
    ds = er500(gp)
    part, _, _ = gp.partition_vertices(ds, G, ps)
    co = gp.make_chunks(ds, K, cs)
    assert np.array_equal(co, ref["chunk_of"])
    opt = gp.TrainOptions(model=gp.ModelConfig(kind=kind, layers=L, hidden=H), epochs=ep, seed=seed, **kw)
    res = gp.train_hybrid(ds, part, co, S, opt)
    met = ref["metrics"].reshape(ep, 5)
    assert np.max(np.abs(res.train_loss - met[:, 1]) / np.abs(met[:, 1])) < 1e-4, (res.train_loss, met[:, 1])
    assert np.max(np.abs(res.metrics[:, 2:5] - met[:, 2:5])) <= 3.0 / (0.2 * ds.num_vertices)
    assert np.array_equal(res.comm.astype(np.uint64), ref["comm"].reshape(ep, 3)), (res.comm, ref["comm"])
    worst, med = 0.0, []
    for l, (W, b) in enumerate(res.params):
        rW = ref[f"W{l}"]
        d = np.abs(W.astype(np.float64) - rW) / np.maximum(np.abs(rW), 1e-3)
        worst = max(worst, float(d.max()))
        med.append(float(np.median(d)))
    assert worst < 2e-3 and max(med) < 1e-4, (worst, med)


def _powerlaw(gp):
    return gp.Dataset.load(os.path.join(GOLD, "powerlaw_2k"))


def test_train_gcn_pipeline_powerlaw_graph(gp):
    """Skewed degrees (Chung-Lu, max degree 822, median 5; tests/golden/make_powerlaw.py): long and
    short rows in one chunk, the degree-ordered rows and dynamic row scheduling."""
    _train_compare(gp, "train_gcn_powerlaw_s2k8", _powerlaw(gp), gp.ModelConfig(kind=0, layers=4, hidden=16), 2, 8,
                   4, 8, 52, fix_alpha=2)


def test_train_hybrid_powerlaw_graph(gp):
    """BASELINE configs[4] in miniature: 2 stages x 2 graph partitions, GCNII, power-law graph."""
    ref = golden("train_gcnii_powerlaw_hyb_s2g2")
    ds = _powerlaw(gp)
    part, _, _ = gp.partition_vertices(ds, 2, 1)
    co = gp.make_chunks(ds, 4, 3)
    assert np.array_equal(co, ref["chunk_of"])
    opt = gp.TrainOptions(model=gp.ModelConfig(kind=2, layers=8, hidden=16), epochs=8, seed=51, fix_alpha=3)
    res = gp.train_hybrid(ds, part, co, 2, opt)
    met = ref["metrics"].reshape(8, 5)
    assert np.max(np.abs(res.train_loss - met[:, 1]) / np.abs(met[:, 1])) < 1e-4, (res.train_loss, met[:, 1])
    assert np.array_equal(res.comm.astype(np.uint64), ref["comm"].reshape(8, 3))
    worst = max(float((np.abs(W.astype(np.float64) - ref[f"W{l}"]) / np.maximum(np.abs(ref[f"W{l}"]), 1e-3)).max())
                for l, (W, _) in enumerate(res.params))
    assert worst < 2e-3, worst


def test_train_gcn16_arxivlike_20_epoch_curve(gp):
    """BASELINE configs[1] in miniature over 20 epochs (the north star's loss-curve horizon): 20 K
    vertices at arxiv-like density, 16-layer GCN, 2 stages x 8 chunks, default staleness. Loss within
    rel 1e-5 every epoch, parameters within the usual bars, ledger exact. The 16-layer GCN's logits stay
    near-uniform for 20 epochs (loss ~ ln 40), so argmax ties flip on rounding: accuracies within 0.2 %.
    Adam moves a weight by ~lr per step whatever the gradient's size, so gradient elements whose sign
    sits at fp32 rounding level (vanishing gradients of the upper layers) can take a few opposite
    steps: weights within 5 lr (5e-3) absolute, median relative 1e-3 (measured: 3.8e-3, <= 3.8e-4;
    lower layers ~1e-5, a param-diff probe, round 1). The engine against itself with only the
    parameter-gradient summation order changed (GP_PGRAD=simt) differs by the same amounts (2.9e-3 at
    layer 14), so this is fp32 amplification, not a semantic difference."""
    ds = gp.Dataset.synthetic_er(20000, 0.0007, 21, 128, 40, 5)
    res = _train_compare(gp, "train_gcn16_arxivlike_s2k8_20ep", ds, gp.ModelConfig(kind=0, layers=16, hidden=64),
                         2, 8, 6, 20, 61, loss_tol=1e-5, acc_tol=2e-3, param_abs_tol=5e-3, fix_alpha=10)
    assert res.metrics.shape[0] == 20


@pytest.mark.parametrize("loops", [True, False], ids=["self_loops", "no_self_loops"])
@pytest.mark.parametrize("K", [3, 64])
def test_device_graph_build_equals_host_builder(gp, loops, K, monkeypatch):
    """k_build_edges (GP_GRAPH_BUILD=device) against the host builder on a sparse graph with
    isolated vertices (rows holding only the self loop, or nothing), self loops on and off, and
    64 chunks (the largest done-set / per-chunk histogram): bit-identical training."""
    ds = gp.Dataset.synthetic_er(700, 0.003, 5, 12, 4, 2)
    off, _, _ = ds.graph()
    assert (np.diff(off) == 0).any()  # isolated vertices present
    co = gp.make_chunks(ds, K, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=4, hidden=16, self_loops=loops)
    opt = gp.TrainOptions(model=model, epochs=4, seed=3, fix_alpha=2)
    runs = {}
    for mode in ("device", "host"):
        monkeypatch.setenv("GP_GRAPH_BUILD", mode)
        runs[mode] = gp.train_pipeline(ds, co, 2, opt)
    np.testing.assert_array_equal(runs["device"].train_loss, runs["host"].train_loss)
    for (Wa, _), (Wb, _) in zip(runs["device"].params, runs["host"].params):
        assert np.array_equal(Wa.view(np.uint32), Wb.view(np.uint32))


@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
@pytest.mark.parametrize("kind", [0, 2], ids=["gcn", "gcnii"])
def test_fused_optimizer_step_equals_per_layer_kernels(gp, optimizer, kind, monkeypatch):
    """k_param_step (one launch: Adam / SGD, W^T, tcgen05 operand preparation for every layer)
    against the per-layer k_adam / k_transpose / k_tc_prep sequence (GP_FUSED_STEP=0), with the
    CUDA-core transforms too (they read W^T): bit-identical training."""
    ds = er500(gp)
    co = gp.make_chunks(ds, 4, 3)
    opt = gp.TrainOptions(model=gp.ModelConfig(kind=kind, layers=5, hidden=16), epochs=5, seed=4, fix_alpha=2,
                          optimizer=optimizer, lr=0.01)
    for tc in ("1", "0"):
        monkeypatch.setenv("GP_TC_XFORM", tc)
        monkeypatch.delenv("GP_FUSED_STEP", raising=False)
        fused = gp.train_pipeline(ds, co, 2, opt)
        monkeypatch.setenv("GP_FUSED_STEP", "0")
        loop = gp.train_pipeline(ds, co, 2, opt)
        np.testing.assert_array_equal(fused.train_loss, loop.train_loss)
        for (Wa, ba), (Wb, bb) in zip(fused.params, loop.params):
            assert np.array_equal(Wa.view(np.uint32), Wb.view(np.uint32))
            assert np.array_equal(ba.view(np.uint32), bb.view(np.uint32))
