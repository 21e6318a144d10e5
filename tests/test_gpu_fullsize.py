"""Parity at the headline size (BASELINE.json configs[2], Reddit shape: 232,965 vertices, 114.6 M
directed edges, F = 602, H = 100): one GCNII epoch on the GPU, then sampled rows recomputed with the
reference's float arithmetic (nn.hpp:143-197: dropped inputs, ascending neighbours, one rounded
multiply and one rounded add per term, GCNII mixes in float) and compared BIT-EXACTLY. The dropout
masks come from the C oracle (DropMask::make, nn.hpp:112-127). Also a whole-graph property: the
aggregation is linear, so the row sums of pre over the first conv layer match A_hat applied to the
row sums of its gather table (fp64, relative 1e-5)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, E2, F, C, H = 232965, 114615892, 602, 41, 100


@pytest.fixture(scope="module", autouse=True)
def need_gpu(gp):
    if gp.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


def _bits(mask_words, rows, cols):
    """keep[r, j] for original rows `rows` from DropMask bits (bit i = v*cols + j)."""
    idx = rows.astype(np.uint64)[:, None] * np.uint64(cols) + np.arange(cols, dtype=np.uint64)[None, :]
    return ((mask_words[idx >> np.uint64(6)] >> (idx & np.uint64(63))) & np.uint64(1)).astype(bool)


def _dense_rows(x, W, b):
    """dense_rows (matrix.hpp:63-74) for many rows at once: y = b; y += x_i * W[i] ascending i."""
    y = np.broadcast_to(b.astype(np.float32), (x.shape[0], W.shape[1])).copy() if b is not None and b.size \
        else np.zeros((x.shape[0], W.shape[1]), np.float32)
    for i in range(W.shape[0]):
        y = y + x[:, i:i + 1] * W[i][None, :]
    return y


def test_reddit_shape_epoch1_rows_bit_exact(gp, monkeypatch):
    monkeypatch.setenv("GP_LEAN", "0")  # activations and gather tables kept apart from dz / dagg
    monkeypatch.setenv("GP_TC_XFORM", "0")  # bit-exact rows need the CUDA-core transforms
    from oracle import oracle as O
    ds = gp.Dataset.synthetic_er(N, E2 / (N * (N - 1)), 1, F, C, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=4, hidden=H, dropout=0.5)
    specs = gp.build_layer_specs(model, F, C)
    params = gp.init_params(model, F, C, 1)
    off, cols, vals = ds.normalize_adjacency(True)
    x, lab, sp = ds.arrays()
    eng = gp.StageEngine(num_vertices=N, num_chunks=1, specs=specs, stage=0, num_stages=1, layer_range=(0, 4),
                         hidden=H, num_classes=C, dropout=0.5, seed=1, device=0)
    eng.upload_graph(off, cols, vals, np.zeros(N, np.uint32))
    eng.upload_features(x)
    eng.upload_labels(lab, sp)
    for l, (W, b) in enumerate(params):
        eng.set_params(l, W, b)
    eng.run_epoch(1, [0])
    h0_gpu = eng.download("h", 0)
    h1_gpu = eng.download("h", 1)
    pre1_gpu = eng.download("pre", 1)
    g1_gpu = eng.download("gather", 1)
    eng.close()

    rng = np.random.default_rng(2308)
    sample = np.sort(rng.choice(N, 48, replace=False)).astype(np.int64)
    nbr = np.unique(np.concatenate([cols[off[v]:off[v + 1]] for v in sample])).astype(np.int64)
    rows = np.union1d(sample, nbr)
    scale = np.float32(2.0)  # T(1 / keep) with keep = 0.5
    m0 = O.dropmask(0.5, 1, 1, 0, N, F)
    m1 = O.dropmask(0.5, 1, 1, 1, N, H)
    # layer 0 (Dense 602 -> 100, ReLU) on every row the sample's aggregation reads
    pre0 = np.where(_bits(m0, rows, F), x[rows] * scale, np.float32(0))
    W0, b0 = params[0]
    h0 = _dense_rows(pre0, W0, b0)
    h0[h0 < 0] = 0
    assert np.array_equal(h0.view(np.uint32), h0_gpu[rows].view(np.uint32)), "layer 0 not bit-exact"
    # layer 1 (Gcn2Conv): dropped gather table, ascending neighbours, GCNII mixes in float
    g1 = np.where(_bits(m1, rows, H), h0 * scale, np.float32(0))
    assert np.array_equal(g1.view(np.uint32), g1_gpu[rows].view(np.uint32)), "gather table not bit-exact"
    pos = {int(v): i for i, v in enumerate(rows)}
    a, beta = np.float32(specs[1].alpha), np.float32(specs[1].beta)
    oma, omb = np.float32(1) - a, np.float32(1) - beta
    W1, _ = params[1]
    for v in sample:
        z = np.zeros(H, np.float32)
        for i in range(int(off[v]), int(off[v + 1])):
            z = z + vals[i] * g1[pos[int(cols[i])]]
        pre = oma * z + a * h0[pos[int(v)]]
        assert np.array_equal(pre.view(np.uint32), pre1_gpu[v].view(np.uint32)), f"pre1 row {v}"
        out = _dense_rows(pre[None, :], W1, None)[0]
        out = omb * pre + beta * out
        out[out < 0] = 0
        assert np.array_equal(out.view(np.uint32), h1_gpu[v].view(np.uint32)), f"h1 row {v}"
    # whole graph: sum_j pre1[v, j] = (1-a) sum_u A[v,u] sum_j g1[u, j] + a sum_j h0[v, j]
    rs_g = g1_gpu.astype(np.float64).sum(1)
    deg = np.diff(off.astype(np.int64))
    agg = np.add.reduceat(vals.astype(np.float64) * rs_g[cols], off[:-1].astype(np.int64)) * (deg > 0)
    want = float(oma) * agg + float(a) * h0_gpu.astype(np.float64).sum(1)
    got = pre1_gpu.astype(np.float64).sum(1)
    assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want))


def test_reddit_shape_64_layer_runs_are_deterministic(gp):
    """The headline configuration (64-layer GCNII, K = 4, 4-stream wavefront, 5-CTA gathers, tcgen05
    parameter gradients) trained twice for 3 epochs gives bit-identical losses and parameters."""
    ds = gp.Dataset.synthetic_er(N, E2 / (N * (N - 1)), 1, F, C, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=64, hidden=H, dropout=0.5)
    co = gp.make_chunks(ds, 4, 1)
    runs = [gp.train_pipeline(ds, co, 1, gp.TrainOptions(model=model, epochs=3, seed=1)) for _ in range(2)]
    assert np.array_equal(runs[0].train_loss, runs[1].train_loss)
    assert np.all(np.isfinite(runs[0].train_loss))
    for (Wa, ba), (Wb, bb) in zip(runs[0].params, runs[1].params):
        assert np.array_equal(Wa.view(np.uint32), Wb.view(np.uint32))


@pytest.mark.parametrize("env", [{}, {"GP_MERGED_G": "0"}, {"GP_REMASK_OVERLAP": "0"}],
                         ids=["wavefront", "wavefront_split_g", "wavefront_remask_in_order"])
def test_reddit_shape_wavefront_equals_serial_chunks(gp, env, monkeypatch):
    """K = 32 (the 8-stage chunk count, where four chunks are in flight on the wavefront streams): the
    wavefront, with split or merged gather tables, trains bit-identically to serial chunks (GP_WAVE=1),
    so no chunk reads a gather row another stream is writing."""
    ds = gp.Dataset.synthetic_er(N, E2 / (N * (N - 1)), 1, F, C, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=16, hidden=H, dropout=0.5)
    co = gp.make_chunks(ds, 32, 1)
    opt = gp.TrainOptions(model=model, epochs=3, seed=1)
    monkeypatch.setenv("GP_WAVE", "1")
    serial = gp.train_pipeline(ds, co, 1, opt)
    monkeypatch.delenv("GP_WAVE")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    wave = gp.train_pipeline(ds, co, 1, opt)
    assert np.array_equal(wave.train_loss, serial.train_loss)
    for (Wa, _), (Wb, _) in zip(wave.params, serial.params):
        assert np.array_equal(Wa.view(np.uint32), Wb.view(np.uint32))


@pytest.mark.parametrize("K", [4, 32])
def test_reddit_shape_filtered_csr_equals_batch_filter(gp, K, monkeypatch):
    """The per-epoch done-filtered backward CSR (default) and the per-batch ballot filter
    (GP_BWD_CSR=0) gather the same entries in the same order: bit-identical training at the
    full Reddit shape, at the 1-GPU and the 8-stage chunk counts."""
    ds = gp.Dataset.synthetic_er(N, E2 / (N * (N - 1)), 1, F, C, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=8, hidden=H, dropout=0.5)
    co = gp.make_chunks(ds, K, 1)
    opt = gp.TrainOptions(model=model, epochs=3, seed=1)
    base = gp.train_pipeline(ds, co, 1, opt)
    monkeypatch.setenv("GP_BWD_CSR", "0")
    batch = gp.train_pipeline(ds, co, 1, opt)
    assert np.array_equal(base.train_loss, batch.train_loss)
    for (Wa, _), (Wb, _) in zip(base.params, batch.params):
        assert np.array_equal(Wa.view(np.uint32), Wb.view(np.uint32))


def test_reddit_shape_device_graph_build_equals_host(gp, monkeypatch):
    """train_pipeline ships the raw neighbour lists and k_build_edges normalises, renumbers and
    packs them on the device (default for large graphs); the host builder (GP_GRAPH_BUILD=host)
    gives the same entries, order and weights: bit-identical training at the Reddit shape."""
    ds = gp.Dataset.synthetic_er(N, E2 / (N * (N - 1)), 1, F, C, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=4, hidden=H, dropout=0.5)
    co = gp.make_chunks(ds, 4, 1)
    opt = gp.TrainOptions(model=model, epochs=2, seed=1)
    dev = gp.train_pipeline(ds, co, 1, opt)
    monkeypatch.setenv("GP_GRAPH_BUILD", "host")
    host = gp.train_pipeline(ds, co, 1, opt)
    assert np.array_equal(dev.train_loss, host.train_loss)
    for (Wa, _), (Wb, _) in zip(dev.params, host.params):
        assert np.array_equal(Wa.view(np.uint32), Wb.view(np.uint32))


@pytest.mark.parametrize("mode", ["device", "host"])
def test_raw_graph_with_self_loop_is_rejected(gp, mode, monkeypatch):
    """A self loop (or an out-of-range neighbour) in the raw lists is rejected by both builders,
    like normalize_adjacency's input check."""
    monkeypatch.setenv("GP_GRAPH_BUILD", mode)
    ds = gp.Dataset.synthetic_er(300, 0.05, 1, 8, 3, 1)
    off, nb, _ = ds.graph()
    nb = nb.copy()
    nb[int(off[5])] = 5  # vertex 5 lists itself
    co = gp.make_chunks(ds, 2, 1)
    specs = gp.build_layer_specs(gp.ModelConfig(kind=gp.ModelKind.GCN, layers=2, hidden=8), 8, 3)
    eng = gp.StageEngine(specs=specs, num_vertices=300, num_chunks=2, stage=0, num_stages=1,
                         layer_range=(0, 2), hidden=8, num_classes=3, dropout=0.5, seed=1)
    with pytest.raises(gp.InvalidArgument):
        eng.upload_graph_raw(off, nb, co, self_loops=True)
    eng.close()
