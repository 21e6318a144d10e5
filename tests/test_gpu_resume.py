"""Checkpoint/resume (extension of the reference's write-only stage checkpoints, nn.hpp:497-531):
parameters + Adam moments + epoch counter restored, epochs continue (dropout keys, chunk order).
In synchronous mode nothing else carries state across epochs, so 3 + 3 resumed epochs equal 6
uninterrupted ones bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ER500 = (500, 0.02, 3, 16, 5, 9)


@pytest.fixture(scope="module", autouse=True)
def need_gpu(gp):
    if gp.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


@pytest.mark.parametrize("kind,S", [("gcnii", 2), ("gcn", 1)])
def test_resume_synchronous_is_exact(gp, tmp_path, kind, S):
    ds = gp.Dataset.synthetic_er(*ER500)
    mk = gp.ModelKind.GCNII if kind == "gcnii" else gp.ModelKind.GCN
    model = gp.ModelConfig(kind=mk, layers=5, hidden=16)
    co = gp.make_chunks(ds, 4, 3)
    base = dict(model=model, seed=7, synchronous_mode=True)
    full = gp.train_pipeline(ds, co, S, gp.TrainOptions(epochs=6, **base))
    state = str(tmp_path / "state.ckpt")
    first = gp.train_pipeline(ds, co, S, gp.TrainOptions(epochs=3, save_state_path=state, **base))
    np.testing.assert_array_equal(first.train_loss, full.train_loss[:3])
    names = [n for n, _ in gp.load_checkpoint(state)]
    assert names[0] == "train.state" and "layer0.weight.adam_m" in names
    second = gp.train_pipeline(ds, co, S, gp.TrainOptions(epochs=3, resume_path=state, **base))
    assert second.metrics[:, 0].tolist() == [4, 5, 6]
    np.testing.assert_array_equal(second.train_loss, full.train_loss[3:])
    for (Wa, ba), (Wb, bb) in zip(second.params, full.params):
        assert np.array_equal(Wa.view(np.uint32), Wb.view(np.uint32))
        if ba is not None and len(ba):
            assert np.array_equal(np.asarray(ba).view(np.uint32), np.asarray(bb).view(np.uint32))


def test_resume_rejects_mismatched_model(gp, tmp_path):
    ds = gp.Dataset.synthetic_er(*ER500)
    co = gp.make_chunks(ds, 2, 3)
    state = str(tmp_path / "s.ckpt")
    gp.train_pipeline(ds, co, 1, gp.TrainOptions(model=gp.ModelConfig(kind=gp.ModelKind.GCN, layers=3, hidden=8),
                                                 epochs=1, save_state_path=state))
    with pytest.raises(gp.InvalidArgument):
        gp.train_pipeline(ds, co, 1, gp.TrainOptions(model=gp.ModelConfig(kind=gp.ModelKind.GCN, layers=3, hidden=16),
                                                     epochs=1, resume_path=state))


def _assert_same(a, b):
    for (Wa, _), (Wb, _) in zip(a.params, b.params):
        assert np.array_equal(Wa.view(np.uint32), Wb.view(np.uint32))


@pytest.mark.parametrize("lean", ["1", "0"])
@pytest.mark.parametrize("case", [
    # kind, S, G, split epoch (fix_alpha 2: t0 = 3 resumes mid-version, t0 = 4 right before a refresh), extras
    ("gcnii", 2, 1, 3, {}),
    ("gcnii", 2, 1, 4, {}),
    ("gcn", 1, 1, 4, {"historical_gradients": True}),
    ("sage", 2, 1, 3, {"historical_gradients": True}),
    ("gcnii", 2, 2, 4, {}),
], ids=["gcnii_s2_t3", "gcnii_s2_t4", "gcn_hist_t4", "sage_hist_s2_t3", "gcnii_hybrid_s2g2_t4"])
def test_resume_stale_mode_is_exact(gp, tmp_path, monkeypatch, case, lean):
    """Default (stale) mode: the saved state holds the historical-embedding rows the next epoch
    reads (h_snap / in_snap / dagg_snap after the snapshot rule, engines_impl.hpp:671-679), so a
    resumed run equals the uninterrupted one bit for bit, on either side of a snapshot refresh."""
    monkeypatch.setenv("GP_LEAN", lean)
    kind, S, G, t0, extra = case
    ds = gp.Dataset.synthetic_er(*ER500)
    mk = {"gcn": gp.ModelKind.GCN, "gcnii": gp.ModelKind.GCNII, "sage": gp.ModelKind.SAGE}[kind]
    model = gp.ModelConfig(kind=mk, layers=5, hidden=16)
    co = gp.make_chunks(ds, 4, 3)
    base = dict(model=model, seed=11, fix_alpha=2, **extra)

    def train(**kw):
        if G == 1:
            return gp.train_pipeline(ds, co, S, gp.TrainOptions(**base, **kw))
        part, _, _ = gp.partition_vertices(ds, G, 2)
        return gp.train_hybrid(ds, part, co, S, gp.TrainOptions(**base, **kw))

    full = train(epochs=7)
    state = str(tmp_path / "state.ckpt")
    train(epochs=t0, save_state_path=state)
    names = [n for n, _ in gp.load_checkpoint(state)]
    assert any(n.startswith("history.") for n in names)
    second = train(epochs=7 - t0, resume_path=state)
    assert second.metrics[:, 0].tolist() == list(range(t0 + 1, 8))
    np.testing.assert_array_equal(second.train_loss, full.train_loss[t0:])
    _assert_same(second, full)


def test_resume_stale_without_history_is_rejected(gp, tmp_path):
    ds = gp.Dataset.synthetic_er(*ER500)
    co = gp.make_chunks(ds, 4, 3)
    model = gp.ModelConfig(kind=gp.ModelKind.GCN, layers=3, hidden=8)
    state = str(tmp_path / "s.ckpt")
    gp.train_pipeline(ds, co, 1, gp.TrainOptions(model=model, epochs=2, synchronous_mode=True, save_state_path=state))
    with pytest.raises(gp.InvalidArgument, match="historical"):
        gp.train_pipeline(ds, co, 1, gp.TrainOptions(model=model, epochs=1, resume_path=state))
