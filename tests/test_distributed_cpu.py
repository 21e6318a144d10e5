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
        ids = D.exchange_unique_ids(dist, rank, world, lambda: os.urandom(128))
        up, down = D.boundary_ids(ids, rank, world)
        if rank > 0:
            assert up == ids[rank - 1]
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
