"""Measured trace (FabricOptions::collect_trace, fabric.cpp:222-264) and the run outputs built on it:
per-chunk compute spans from CUDA events on one %globaltimer timebase, the reference's event
kinds and order, bubble_analysis (analytics.cpp:59-86) over real device time."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ER500 = (500, 0.02, 3, 16, 5, 9)


@pytest.fixture(scope="module", autouse=True)
def need_gpu(gp):
    if gp.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


@pytest.mark.parametrize("model_kind,S,K", [("gcn", 2, 4), ("gcnii", 3, 6)])
def test_trace_structure_and_bubble(gp, tmp_path, model_kind, S, K):
    ds = gp.Dataset.synthetic_er(*ER500)
    kind = gp.ModelKind.GCN if model_kind == "gcn" else gp.ModelKind.GCNII
    model = gp.ModelConfig(kind=kind, layers=6, hidden=16)
    co = gp.make_chunks(ds, K, 3)
    T = 3
    base = gp.train_pipeline(ds, co, S, gp.TrainOptions(model=model, epochs=T, seed=5, fix_alpha=2))
    res = gp.train_pipeline(ds, co, S, gp.TrainOptions(model=model, epochs=T, seed=5, fix_alpha=2,
                                                       collect_trace=True))
    # tracing runs chunks serially: same arithmetic, same results
    np.testing.assert_array_equal(res.train_loss, base.train_loss)
    assert len(base.trace) == 0
    tr = res.trace
    assert len(tr) > 0
    assert np.all(tr["t_end"] >= tr["t_start"]) and tr["t_start"].min() == 0.0
    assert np.all(np.diff(tr["t_start"]) >= 0)  # sorted by start (then worker)
    ranges = gp.make_stage_assignment(6, S)
    for w in range(S):
        ev = tr[tr["worker"] == w]
        comp = ev[ev["kind"] == 0]
        # per epoch: K forward + K backward chunk spans + the parameter step
        assert len(comp) == T * (2 * K + 1)
        assert np.all(comp["layer_lo"] == ranges[w][0]) and np.all(comp["layer_hi"] == ranges[w][1] - 1)
        # a stage's compute spans never overlap
        c = np.sort(comp, order="t_start")
        assert np.all(c["t_start"][1:] >= c["t_end"][:-1] - 1e-9)
        nsend = (ev["kind"] == 1).sum()
        nrecv = (ev["kind"] == 2).sum()
        assert nsend == T * K * ((w < S - 1) + (w > 0))
        assert nrecv == nsend and (ev["kind"] == 3).sum() == nrecv
        assert sorted(set(comp["chunk"].tolist())) == [-1] + list(range(K))
    # every forward message is received no earlier than it was sent; each stage anchors its events to
    # %globaltimer with one stamp kernel per epoch, so cross-stage times carry a few microseconds of
    # anchor jitter (50 us tolerance)
    for w in range(1, S):
        sends = tr[(tr["worker"] == w - 1) & (tr["kind"] == 1)]
        recvs = tr[(tr["worker"] == w) & (tr["kind"] == 2)]
        for k in range(K):
            assert recvs[recvs["chunk"] == k]["t_start"].min() >= sends[sends["chunk"] == k]["t_start"].min() - 5e-5
    b = gp.bubble_analysis(tr)
    assert b["stages"] == S and b["chunks"] == K
    assert b["ideal_bubble"] == pytest.approx((S - 1) / (K + S - 1))
    assert 0.0 <= b["measured_bubble"] < 1.0
    assert np.all((res.metrics[:, 6] >= 0) & (res.metrics[:, 6] < 1))
    if S > 1:  # per-epoch measured idle fraction (engines_impl.hpp:887-891): stage 1 waits for chunk 0
        assert np.all(res.metrics[:, 6] > 0)
    gp.write_run_outputs(res, str(tmp_path))
    assert sum(1 for _ in open(tmp_path / "trace.jsonl")) == len(tr)
    assert open(tmp_path / "metrics.csv").read().count("\n") == T + 1
    pipe = res.ledger[:, 0:2, :].sum()
    assert pipe == res.comm[:, 1].sum()


@pytest.mark.parametrize("mode", ["sync", "hybrid"])
def test_trace_sync_and_hybrid(gp, mode):
    """Synchronous mode traces one whole-partition compute span per direction (chunk -1,
    engines_impl.hpp:811, :867); hybrid workers trace like stages (G workers per stage)."""
    ds = gp.Dataset.synthetic_er(*ER500)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=5, hidden=16)
    co = gp.make_chunks(ds, 4, 3)
    T = 2
    if mode == "sync":
        res = gp.train_pipeline(ds, co, 2, gp.TrainOptions(model=model, epochs=T, seed=3, synchronous_mode=True,
                                                           collect_trace=True))
        W = 2
    else:
        part, _, _ = gp.partition_vertices(ds, 2, 1)
        res = gp.train_hybrid(ds, part, co, 2, gp.TrainOptions(model=model, epochs=T, seed=3, fix_alpha=2,
                                                                collect_trace=True))
        W = 4
    tr = res.trace
    assert sorted(set(tr["worker"].tolist())) == list(range(W))
    for w in range(W):
        comp = tr[(tr["worker"] == w) & (tr["kind"] == 0)]
        per_epoch = 3 if mode == "sync" else 2 * 4 + 1  # fwd, bwd, param step | per chunk + step
        assert len(comp) == T * per_epoch, (w, len(comp))
        c = np.sort(comp, order="t_start")
        assert np.all(c["t_start"][1:] >= c["t_end"][:-1] - 1e-9)
    b = gp.bubble_analysis(tr)
    assert 0.0 <= b["measured_bubble"] < 1.0


def test_train_tool_writes_reference_run_outputs(gp, tmp_path):
    """tools/gnnpipe_train.py: the reference CLI's run outputs from the engine, then a resumed run."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "gnnpipe_train", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools",
                                      "gnnpipe_train.py"))
    tool = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(tool)
    out = tmp_path / "run"
    args = ["--synthetic", "er:500:0.02:3:16:5:9", "--model", "gcnii", "--layers", "5", "--hidden", "16",
            "--stages", "2", "--epochs", "3", "--trace", "--out", str(out)]
    tool.main(args)
    for name in ("metrics.csv", "trace.jsonl", "comm_report.csv", "stage_0.ckpt", "stage_1.ckpt", "state.ckpt",
                 "chunks.txt"):
        assert (out / name).exists(), name
    k, co = gp.load_assignment(str(out / "chunks.txt"))
    ds = gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)
    assert k == 8 and np.array_equal(co, gp.make_chunks(ds, 8, 1))
    assert open(out / "metrics.csv").read().count("\n") == 4
    names = [n for n, _ in gp.load_checkpoint(str(out / "stage_1.ckpt"))]
    assert names[0].startswith("layer") and names[0].endswith(".weight")
    tool.main(args[:-2] + ["--resume", str(out / "state.ckpt"), "--chunks-file", str(out / "chunks.txt"),
                           "--out", str(tmp_path / "run2")])
    assert open(tmp_path / "run2" / "metrics.csv").read().splitlines()[1].startswith("4,")
    assert open(tmp_path / "run2" / "chunks.txt").read() == open(out / "chunks.txt").read()
