"""Multi-process host logic of the N>1 pipeline, on CPU with gloo (world_size 2 and 4).

Each rank plays one pipeline stage: it builds the same dataset and chunk plan (must be
identical across ranks), receives the stage-boundary ids from rank 0, derives its message
schedule, and checks against its neighbours that every send meets a matching recv in the
same order, that the summed ledger equals the closed form 2(S-1)*N*H*vecs*4
(analytics.cpp:12-15), and that max-over-ranks timing works.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sync, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2308_10087_b200 as gp
        from paper_2308_10087_b200 import distributed as D
        S, K, H = world, 4 * world, 16
        ds = gp.Dataset.synthetic_er(400, 0.03, 2, 12, 5, 2)
        chunk_of = gp.make_chunks(ds, K, 7)
        # identical host prep on every rank (bit-exact chunking)
        allc = [None] * world
        dist.all_gather_object(allc, chunk_of.tobytes())
        assert all(c == allc[0] for c in allc)
        # NCCL stage-boundary ids: the engine's own gp_nccl_unique_id on rank 0 (works without a GPU)
        ids = D.exchange_unique_ids(dist, rank, world, gp.nccl_unique_id)
        assert len(ids) == world - 1 and all(len(i) == 128 and any(i) for i in ids)
        up, down = D.boundary_ids(ids, rank, world)
        if rank > 0:
            assert up == ids[rank - 1]
        if rank < world - 1:
            assert down == ids[rank]
        # CUDA-IPC link setup: every stage's (up, down) export blobs meet their neighbours'
        blob = lambda tag: bytes([rank, tag]) + bytes(gp.IPC_BLOB_BYTES - 2)
        mine = (blob(1) if rank > 0 else None, blob(2) if rank < world - 1 else None)
        up_peer, down_peer = D.exchange_ipc_blobs(dist, rank, world, mine)
        assert (up_peer[:2] == bytes([rank - 1, 2])) if rank > 0 else up_peer is None
        assert (down_peer[:2] == bytes([rank + 1, 1])) if rank < world - 1 else down_peer is None
        # hybrid group link setup: 2 groups of world/2 workers exchange their group blobs
        if world % 2 == 0:
            G = world // 2
            st, gr = rank // G, rank % G
            peers = D.exchange_group_blobs(dist, st, gr, G, bytes([st, gr]) * 8)
            assert all(peers[r] == bytes([st, r]) * 8 for r in range(G))  # group-rank order, own included
        # schedule agreement with neighbours, for 3 epochs of shuffled orders
        L = 8
        model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=L, hidden=H)
        specs = gp.build_layer_specs(model, 12, 5)
        lo, hi = D.stage_ranges(L, S)[rank]
        assert (lo, hi) == gp.make_stage_assignment(L, S)[rank]
        rows = np.bincount(chunk_of, minlength=K)
        tot = 0
        for t in range(1, 4):
            order = [int(k) for k in gp.shuffle_chunk_order(K, t, 1)]
            mine = D.message_schedule(order, rank, S, sync)
            sched = [None] * world
            dist.all_gather_object(sched, mine)
            for s in range(world - 1):
                sends = [k for op, k in sched[s] if op == "send_fwd"]
                recvs = [k for op, k in sched[s + 1] if op == "recv_fwd"]
                assert sends == recvs
                sends_b = [k for op, k in sched[s + 1] if op == "send_bwd"]
                recvs_b = [k for op, k in sched[s] if op == "recv_bwd"]
                assert sends_b == recvs_b
            f, b = D.stage_ledger(order, rank, S, rows, specs[hi - 1].out_dim, specs[lo].in_dim, h0_width=H, sync=sync)
            tot += f + b
        t_all = torch_sum(tot)
        want = 3 * 2 * (S - 1) * ds.num_vertices * H * 4 * 2
        assert t_all == want, (t_all, want)
        assert D.max_over_ranks(dist, float(rank)) == float(world - 1)
        # every rank plans its stage's device memory with the engine's layout pass (no GPU)
        plan = gp.stage_footprint(nnz_norm=1 << 20, num_features=12, specs=specs, num_vertices=ds.num_vertices,
                                  num_chunks=K, stage=rank, num_stages=S, layer_range=(lo, hi), hidden=H,
                                  num_classes=5, dropout=0.5, seed=1)
        allp = [None] * world
        dist.all_gather_object(allp, plan)
        assert all(x > 0 for x in allp) and (world < 3 or len(set(allp[1:-1])) == 1)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def torch_sum(x):
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t)
    return int(t.item())


@pytest.mark.parametrize("world,sync", [(2, False), (2, True), (4, False)])
def test_pipeline_plumbing_gloo(world, sync):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sync, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, "ok") for r in range(world)], res


def test_schedule_single_stage_has_no_messages():
    from paper_2308_10087_b200 import distributed as D
    assert D.message_schedule([2, 0, 1], 0, 1) == []


def test_bench_self_launches_ranks_on_cpu():
    """bench.py --gpus 2 without WORLD_SIZE relaunches itself under torchrun with 2 ranks; on the
    reference arm rank 0 alone prints the line (S = 2 stage threads) and rank 1 exits 0."""
    import json
    import subprocess
    import sys
    from oracle.blob import have_ref
    if not have_ref():
        pytest.skip("oracle/_ref/ref_driver not built")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference", "--workload", "er4k",
                        "--steps", "2", "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["config"]["stages"] == 2
    assert lines[0]["config"]["chunks"] == 8
