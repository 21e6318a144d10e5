"""Run outputs and analytics against the reference (tests/golden/analytics.npz, produced by the
unmodified reference's bubble_analysis / crossover_report / writers via oracle/ref_driver analytics):
analytics.cpp:12-103, fabric.cpp:136-182, engines.cpp:23-38. Host-only: no GPU needed."""
import os

import numpy as np
import pytest

import paper_2308_10087_b200 as gp

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(HERE, "golden", "analytics.npz")))


def test_bubble_analysis_matches_reference(gold):
    b = gp.bubble_analysis(gold["events"])
    ref = gold["bubble"]
    assert b["measured_bubble"] == ref[0]
    assert b["ideal_bubble"] == ref[1]
    assert (b["stages"], b["chunks"]) == (int(ref[2]), int(ref[3]))
    assert b["span"] == ref[4]


def test_bubble_analysis_rejects_empty_trace():
    with pytest.raises(gp.InvalidArgument):
        gp.bubble_analysis(np.zeros(0, gp.TRACE_DTYPE))


def _inputs(alpha):
    g = gp.CommModelInput(n=232965, layers=64, hidden=100, ways=8, alpha=alpha)
    p = gp.CommModelInput(n=232965, layers=64, hidden=100, stages=8, vecs=2)
    h = gp.CommModelInput(n=232965, layers=64, hidden=100, stages=4, ways=2, alpha=alpha / 3, vecs=2)
    return g, p, h


def test_volumes_and_crossover_match_reference(gold):
    lines = bytes(gold["crossover"]).decode().strip().split("\n")
    for i, alpha in enumerate((0.0, 0.35, 2.5)):
        g, p, h = _inputs(alpha)
        r = gp.crossover_report(g, p, h)
        np.testing.assert_array_equal([r["bytes_graph"], r["bytes_pipeline"], r["bytes_hybrid"]],
                                      gold["volumes"][3 * i:3 * i + 3])
        v = gp.comm_volumes(**{k: getattr(h, k) for k in ("n", "layers", "hidden", "stages", "ways", "alpha",
                                                            "vecs")})
        assert v["hybrid"] == gold["volumes"][3 * i + 2]
        winner, tie, order, *ineq = lines[i].split("|")
        assert r["winner"] == winner and r["tie"] == (tie == "tie")
        assert r["ordering"] == order.rstrip(",").split(",")
        assert r["inequalities"] == ineq


def test_writers_match_reference_bytes(gold, tmp_path):
    # trace.jsonl of the same events
    res = gp.TrainResult(metrics=np.zeros((0, 7)), comm=np.zeros((0, 3), np.uint64), params=[], profile={},
                         peak_buffer_bytes=0, trace=gold["events"], ledger=np.zeros((0, 6, 2), np.uint64))
    # metrics / ledger rows of ref_driver cmd_analytics
    T = 3
    met = np.zeros((T, 7))
    comm = np.zeros((T, 3), np.uint64)
    for e in range(1, T + 1):
        met[e - 1] = [e, 3.7 / e, 0.1 * e, 0.09 * e, 0.08 * e, 0.4 + e * 1e-3, 0.18 / e]
        comm[e - 1] = [11 * e, 373000000 * e, 7 * e]
    led = np.zeros((T, 6, 2), np.uint64)
    for e in range(T):
        for t in range(6):
            for l in range(2):
                if ((e + 1) * 1000003 * (t + 1) + l * 77) % 5:
                    led[e, t, l] = (e + 1) * 123456789 * (t + 1) + l
    res.metrics, res.comm, res.ledger = met, comm, led
    gp.write_run_outputs(res, str(tmp_path))
    for name in ("trace.jsonl", "metrics.csv", "comm_report.csv"):
        assert (tmp_path / name).read_text() == str(gold["file_" + name.replace(".", "_")]), name
    gp.write_compare_csv(str(tmp_path / "compare.csv"), [
        dict(mode="pipeline", n=232965, layers=64, hidden=100, stages=8, ways=1, alpha=0, vecs=2,
             predicted_bytes=2.6e9, measured_bytes=2600000123, rel_error=4.7e-8),
        dict(mode="graph", n=1000, layers=4, hidden=16, stages=1, ways=3, alpha=0.25, vecs=1,
             predicted_bytes=128000, measured_bytes=127990, rel_error=7.8125e-5)])
    assert (tmp_path / "compare.csv").read_text() == str(gold["file_compare_csv"])


def test_train_tool_compare_rows(tmp_path):
    """`gnnsim compare` rows (gnnsim.cpp:305-347) from a result's ledger: graph mode predicts
    2 alpha N sum(in_dim of aggregating layers) 4 bytes, pipeline volume_pipeline, hybrid both."""
    import sys
    from types import SimpleNamespace
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import gnnpipe_train
    ds = gp.Dataset.synthetic_er(200, 0.05, 3, 24, 5, 4)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=4, hidden=16)
    specs = gp.build_layer_specs(model, ds.num_features, ds.num_classes)
    alpha = 0.75
    halo = 2.0 * sum(alpha * 200 * s.in_dim * 4.0 for s in specs if s.aggregates)
    pipe = gp.comm_volumes(200, 4, 16, 2, 2, alpha, 2)["pipeline"]
    comm = np.array([[int(halo), int(pipe), 0], [int(halo) + 40, int(pipe), 0]], np.uint64)
    res = SimpleNamespace(metrics=np.zeros((2, 7)), comm=comm)
    path = str(tmp_path / "compare.csv")
    gnnpipe_train.write_compare(path, "hybrid", ds, model, res, 2, 2, alpha)
    lines = open(path).read().splitlines()
    assert lines[0] == "mode,N,L,H,S,W,alpha,vecs,predicted_bytes,measured_bytes,rel_error"
    assert len(lines) == 3 and all(l.startswith("hybrid,200,4,16,2,2,0.75,2,") for l in lines[1:])
    assert lines[1].endswith(",0")
    assert float(lines[2].split(",")[-1]) == pytest.approx(40 / (halo + pipe))
