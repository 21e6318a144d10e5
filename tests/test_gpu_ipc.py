"""One process per stage over the CUDA-IPC transport (gp_ipc_export / gp_link_ipc).

The in-process pipeline (train_pipeline: stage threads, local D2D links) is the
ground truth here — it is itself pinned to the reference by test_gpu_parity.py —
and the cross-process run must reproduce it BIT-EXACTLY: the transport only moves
rows, it never changes an operation. The box has one GPU, so all stage processes
share device 0 (cudaIpcOpenMemHandle works between processes on one device); on an
8-GPU node the same code pushes over NVLink.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import ipc_stage_worker as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def need_gpu(gp):
    if gp.device_count() == 0:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def in_process(gp, S, epochs):
    ds, model, chunk_of = W.problem()
    res = gp.train_pipeline(ds, chunk_of, S, gp.TrainOptions(model=model, epochs=epochs, seed=1))
    x, lab, sp = ds.arrays()
    return res, float((sp == 1).sum())


def check_same(res, n_train, losses, params):
    assert len(losses) == len(res.train_loss)
    np.testing.assert_allclose(np.asarray(losses) / n_train, res.train_loss, rtol=1e-12, atol=0)
    for l, (Wr, br) in enumerate(res.params):
        assert np.array_equal(params[l][0].view(np.uint32), Wr.view(np.uint32)), f"W{l} differs"
        if br.size:
            assert np.array_equal(params[l][1].view(np.uint32), br.view(np.uint32)), f"b{l} differs"


@pytest.mark.parametrize("S", [2, 3])
def test_ipc_stage_processes_match_in_process_pipeline(gp, tmp_path, S):
    epochs = 12  # crosses the fix_alpha=10 snapshot at t=11
    out = str(tmp_path / "ipc.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={S}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(HERE, "ipc_stage_worker.py"),
           out, str(epochs)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    z = np.load(out)
    res, n_train = in_process(gp, S, epochs)
    L = len(res.params)
    check_same(res, n_train, z["losses"], [(z[f"W{l}"], z[f"b{l}"]) for l in range(L)])


def test_ipc_refuses_stages_sharing_a_context(gp):
    """Two IPC-linked stages of one process on one device would share a CUDA context, where
    an implicit context synchronisation on one stage's thread can wait forever on the other
    stage's pending in-stream wait. gp_link_ipc refuses that pairing (gp_link_local is the
    in-process transport); the same-process, other-device UVA path needs a second GPU."""
    S = 2
    ds, model, chunk_of = W.problem()
    engs = [W.stage_engine(ds, model, chunk_of, r, S, 0) for r in range(S)]
    blobs = [e.ipc_export() for e, _ in engs]
    with pytest.raises(gp.InvalidArgument, match="gp_link_local"):
        engs[0][0].link_ipc(None, blobs[1][0])
    with pytest.raises(gp.InvalidArgument, match="gp_link_local"):
        engs[1][0].link_ipc(blobs[0][1], None)
    for e, _ in engs:
        e.close()
    # ledger: the IPC transport accounts the same bytes as the reference fabric (4 B/value)
    for e, _ in engs:
        e.close()


def test_ipc_link_errors(gp):
    ds, model, chunk_of = W.problem()
    specs = gp.build_layer_specs(model, W.F, W.CLASSES)
    e0 = gp.StageEngine(num_vertices=W.N, num_chunks=W.K, specs=specs, stage=0, num_stages=2, layer_range=(0, 4),
                        hidden=W.H, num_classes=W.CLASSES, dropout=0.5, seed=1)
    with pytest.raises(gp.InvalidArgument, match="upload the graph"):
        e0.ipc_export()
    e0.close()
    a, _ = W.stage_engine(ds, model, chunk_of, 0, 3, 0)
    b, _ = W.stage_engine(ds, model, chunk_of, 1, 3, 0)
    c, _ = W.stage_engine(ds, model, chunk_of, 2, 3, 0)
    ba, bb, bc = a.ipc_export(), b.ipc_export(), c.ipc_export()
    assert ba[0] is None and bc[1] is None and len(bb[0]) == gp.IPC_BLOB_BYTES
    with pytest.raises(gp.InvalidArgument, match="does not face"):
        c.link_ipc(ba[1], None)  # stage 0's blob offered to stage 2
    with pytest.raises(gp.InvalidArgument, match="not an IPC blob"):
        b.link_ipc(bytes(gp.IPC_BLOB_BYTES), None)
    for e in (a, b, c):
        e.close()


HYB_IPC = [
    # kind, L, H, S, G, K, chunk seed, part seed, epochs, seed, staleness
    dict(kind=2, L=5, H=16, S=1, G=2, K=4, cs=3, ps=2, epochs=6, seed=43, fix_alpha=3),
    dict(kind=0, L=4, H=16, S=2, G=2, K=4, cs=3, ps=1, epochs=5, seed=42, fix_alpha=3),
    dict(kind=2, L=5, H=16, S=1, G=3, K=3, cs=5, ps=3, epochs=4, seed=44, sync=True),
    dict(kind=0, L=6, H=12, S=2, G=2, K=6, cs=7, ps=4, epochs=4, seed=45, fix_alpha=2, hist=True),
    dict(kind=1, L=4, H=16, S=2, G=2, K=4, cs=3, ps=1, epochs=4, seed=48, fix_alpha=3),
    # BASELINE configs[4]'s shape in miniature: 4 stages x 2 graph partitions (8 worker
    # processes), GCNII, K = 16, power-law graph
    dict(kind=2, L=8, H=16, S=4, G=2, K=16, cs=3, ps=1, epochs=4, seed=51, fix_alpha=3, data="powerlaw"),
]


@pytest.mark.parametrize("case", HYB_IPC, ids=[f"k{c['kind']}_s{c['S']}g{c['G']}{'_hist' if c.get('hist') else ''}"
                                               f"{'_' + c['data'] if c.get('data') else ''}" for c in HYB_IPC])
def test_ipc_hybrid_processes_match_in_process_hybrid(gp, tmp_path, case):
    """S x G worker processes (gp_link_group_ipc + gp_link_ipc) == train_hybrid in one
    process (gp_link_group + gp_link_local), bit for bit."""
    import json
    out = str(tmp_path / "hyb.npz")
    W = case["S"] * case["G"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(HERE, "ipc_hybrid_worker.py"),
           out, json.dumps(case)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    z = np.load(out)
    import ipc_hybrid_worker as HW
    ds = HW.dataset(case)
    part, _, _ = gp.partition_vertices(ds, case["G"], case["ps"])
    co = gp.make_chunks(ds, case["K"], case["cs"])
    kw = {}
    if "fix_alpha" in case:
        kw["fix_alpha"] = case["fix_alpha"]
    if case.get("hist"):
        kw["historical_gradients"] = True
    if case.get("sync"):
        kw["synchronous_mode"] = True
    opt = gp.TrainOptions(model=gp.ModelConfig(kind=case["kind"], layers=case["L"], hidden=case["H"]),
                          epochs=case["epochs"], seed=case["seed"], **kw)
    res = gp.train_hybrid(ds, part, co, case["S"], opt)
    x, lab, sp = ds.arrays()
    np.testing.assert_allclose(z["loss_sum"] / float((sp == 1).sum()), res.train_loss, rtol=1e-12, atol=0)
    for l, (Wr, br) in enumerate(res.params):
        assert np.array_equal(z[f"W{l}"].view(np.uint32), Wr.view(np.uint32)), f"W{l} differs"
        if br.size:
            assert np.array_equal(z[f"b{l}"].view(np.uint32), br.view(np.uint32)), f"b{l} differs"


def test_group_link_errors(gp):
    ds = gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)
    model = gp.ModelConfig(kind=0, layers=3, hidden=8)
    specs = gp.build_layer_specs(model, ds.num_features, ds.num_classes)
    part, _, _ = gp.partition_vertices(ds, 2, 1)
    co = gp.make_chunks(ds, 2, 1)
    off, cols, vals = ds.normalize_adjacency(True)

    def member(r, G=2):
        e = gp.StageEngine(num_vertices=ds.num_vertices, num_chunks=2, specs=specs, stage=0, num_stages=1,
                           layer_range=(0, 3), hidden=8, num_classes=ds.num_classes, dropout=0.5, seed=1,
                           group_size=G, group_rank=r)
        if G > 1:
            e.upload_partition(part)
        e.upload_graph(off, cols, vals, co)
        return e

    solo = member(0, G=1)
    with pytest.raises(gp.InvalidArgument, match="not a hybrid worker"):
        solo.group_export()
    a, b = member(0), member(1)
    ba, bb = a.group_export(), b.group_export()
    with pytest.raises(gp.InvalidArgument, match="does not match"):
        a.link_group_ipc([None, ba])  # rank 0's own blob offered as rank 1
    with pytest.raises(gp.InvalidArgument, match="not a group blob"):
        a.link_group_ipc([None, bytes(len(bb))])
    for e in (solo, a, b):
        e.close()
