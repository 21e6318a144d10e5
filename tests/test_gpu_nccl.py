"""The NCCL stage transport (gp_link_nccl: one 2-rank communicator per stage boundary,
grouped ncclSend / ncclRecv of a chunk's rows, engines_impl.hpp:690-724 -> fabric.cpp:288-359)
on a one-GPU box: its handshake and error paths. Communicators are created non-blocking and
polled under a watchdog (GP_NCCL_TIMEOUT), so a peer that never joins, or NCCL refusing two
ranks on one device, is an error within the timeout, never a hang. On a multi-GPU node the same
calls run the pipeline (bench.py --gpus N --transport nccl); when NCCL does accept the two
ranks here, the run must equal the in-process pipeline bit for bit."""
import json
import os
import subprocess
import sys
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module", autouse=True)
def need_gpu(gp):
    if gp.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


def engine(gp, stage, S):
    ds = gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)
    model = gp.ModelConfig(kind=gp.ModelKind.GCN, layers=4, hidden=16)
    specs = gp.build_layer_specs(model, ds.num_features, ds.num_classes)
    rng = gp.make_stage_assignment(4, S)[stage]
    return gp.StageEngine(num_vertices=ds.num_vertices, num_chunks=4, specs=specs, stage=stage, num_stages=S,
                          layer_range=rng, hidden=16, num_classes=ds.num_classes, dropout=0.5, seed=1)


def test_unique_id_and_single_stage(gp):
    uid = gp.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    e = engine(gp, 0, 1)
    with pytest.raises(gp.InvalidArgument):
        e.link_nccl(None, uid)
    e.close()


def test_missing_peer_times_out(gp, monkeypatch):
    monkeypatch.setenv("GP_NCCL_TIMEOUT", "5")
    e = engine(gp, 0, 2)
    t0 = time.time()
    with pytest.raises((gp.FabricError, gp.GpuEngineError)):
        e.link_nccl(None, gp.nccl_unique_id())
    assert time.time() - t0 < 60
    e.close()


def test_two_stage_processes_on_one_device(gp, tmp_path):
    idf = str(tmp_path / "nccl.id")
    env = dict(os.environ, GP_NCCL_TIMEOUT="30")
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "nccl_stage_worker.py"), str(s), idf,
                               str(tmp_path / f"out{s}.json")], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for s in (0, 1)]
    for p in procs:
        _, err = p.communicate(timeout=240)
        assert p.returncode == 0, err[-3000:]
    out = [json.load(open(tmp_path / f"out{s}.json")) for s in (0, 1)]
    if all(o.get("linked") and "error" not in o for o in out):
        # NCCL accepted both ranks on one device: the run equals the in-process pipeline
        ds = gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)
        model = gp.ModelConfig(kind=gp.ModelKind.GCN, layers=4, hidden=16)
        res = gp.train_pipeline(ds, gp.make_chunks(ds, 4, 3), 2, gp.TrainOptions(model=model, epochs=3, seed=1))
        n_train = float((ds.arrays()[2] == 1).sum())
        np.testing.assert_allclose(np.asarray(out[1]["losses"]) / n_train, res.train_loss, rtol=1e-12, atol=0)
        got = out[0]["params"] + out[1]["params"]
        for l, (W, _) in enumerate(res.params):
            assert np.array_equal(np.asarray(got[l], np.float32).view(np.uint32), W.view(np.uint32))
    else:  # refused (two ranks on one GPU): a prompt, reported error on both sides
        for o in out:
            assert "error" in o and o["seconds"] < 60, o
