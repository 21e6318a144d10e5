"""The run-output tool (`tools/gnnpipe_train.py`, the reference's `gnnsim train/compare`,
gnnsim.cpp:278-359) on the GPU: every trainer mode, compare.csv against the analytic volumes."""
import csv
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.mark.parametrize("args", [["--mode", "graph", "--workers", "4"],
                                  ["--mode", "pipeline", "--stages", "2"],
                                  ["--mode", "hybrid", "--stages", "2", "--parts", "2"],
                                  ["--mode", "sequential"]],
                         ids=["graph", "pipeline", "hybrid", "sequential"])
def test_train_tool_compare(gp, tmp_path, args, capsys):
    import gnnpipe_train
    out = str(tmp_path / "run")
    gnnpipe_train.main(["--synthetic", "er:500:0.02:3:32:5:4", "--model", "gcnii", "--layers", "4",
                        "--hidden", "16", "--epochs", "3", "--compare", "--out", out] + args)
    for f in ("metrics.csv", "comm_report.csv", "compare.csv", "state.ckpt", "stage_0.ckpt"):
        assert os.path.exists(os.path.join(out, f)), f
    with open(os.path.join(out, "compare.csv")) as fh:
        rows = list(csv.DictReader(fh))
    assert len(rows) == 3
    mode = args[1]
    for r in rows:
        assert r["mode"] == mode
        if mode == "sequential":  # no analytic volume: measured bytes are reported as the error
            assert float(r["measured_bytes"]) == 0
        else:
            assert float(r["measured_bytes"]) > 0
            # the ledger moves exactly the analytic volume (test_analytics.cpp closed forms)
            assert float(r["rel_error"]) < 1e-9, r
