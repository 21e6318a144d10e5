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
