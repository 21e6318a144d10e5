"""Checkpoint files against the reference (tests/golden/checkpoints.npz: files written by the
unmodified reference's save_stage_checkpoint, nn.hpp:511-531 / nn.cpp:82-102). Host-only."""
import os

import numpy as np
import pytest

import paper_2308_10087_b200 as gp

HERE = os.path.dirname(os.path.abspath(__file__))
KINDS = {"ckpt_gcnii": gp.ModelKind.GCNII, "ckpt_gcn_stage1": gp.ModelKind.GCN}


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(HERE, "golden", "checkpoints.npz")))


@pytest.mark.parametrize("name", sorted(KINDS))
def test_stage_checkpoint_bytes_match_reference(gold, tmp_path, name):
    L, H, F, Cc, seed, lo, hi = (int(x) for x in gold[name + "_args"])
    model = gp.ModelConfig(kind=KINDS[name], layers=L, hidden=H)
    params = gp.init_params(model, F, Cc, seed)
    path = str(tmp_path / "s.ckpt")
    gp.save_stage_checkpoint(path, model, F, Cc, params, lo, hi)
    assert np.array_equal(np.fromfile(path, np.uint8), gold[name])


@pytest.mark.parametrize("name", sorted(KINDS))
def test_load_reference_checkpoint(gold, tmp_path, name):
    L, H, F, Cc, seed, lo, hi = (int(x) for x in gold[name + "_args"])
    path = str(tmp_path / "ref.ckpt")
    gold[name].tofile(path)
    tensors = gp.load_checkpoint(path)
    params = gp.init_params(gp.ModelConfig(kind=KINDS[name], layers=L, hidden=H), F, Cc, seed)
    expect = []
    for l in range(lo, hi):
        W, b = params[l]
        expect.append((f"layer{l}.weight", W))
        if b is not None and len(b):
            expect.append((f"layer{l}.bias", np.asarray(b).reshape(1, -1)))
    assert [n for n, _ in tensors] == [n for n, _ in expect]
    for (n, got), (_, want) in zip(tensors, expect):
        assert got.shape == want.shape and np.array_equal(got.view(np.uint32), np.asarray(want, np.float32).view(np.uint32)), n


def test_truncated_checkpoint_raises(gold, tmp_path):
    path = str(tmp_path / "t.ckpt")
    gold["ckpt_gcnii"][:-5].tofile(path)
    with pytest.raises(gp.GnnsimError):
        gp.load_checkpoint(path)


def test_header_escapes_decode_like_the_reference(gp, tmp_path):
    """The header is JSON (nlohmann::json, nn.cpp:104-124): short escapes (\\t, \\b, ...) and
    \\uXXXX code points, incl. surrogate pairs, decode to the same UTF-8 names."""
    import json
    import struct

    import numpy as np
    names = ["tab\there", "café", "smile\U0001F600", "bs\bff\f"]
    header = json.dumps({"tensors": [{"cols": 1, "name": n, "rows": 1} for n in names]},
                        separators=(",", ":"), ensure_ascii=True).encode()
    p = tmp_path / "esc.ckpt"
    p.write_bytes(struct.pack("<Q", len(header)) + header + np.arange(4, dtype=np.float32).tobytes())
    got = gp.load_checkpoint(str(p))
    assert [n for n, _ in got] == names
    assert [float(a[0, 0]) for _, a in got] == [0.0, 1.0, 2.0, 3.0]
