"""One hybrid worker (stage s, partition rank r) per process over CUDA IPC.

Launched by tests/test_gpu_ipc.py as
    python -m torch.distributed.run --nproc-per-node S*G --master-addr 127.0.0.1 \
        --master-port P tests/ipc_hybrid_worker.py OUT.npz JSON_CASE
Worker w runs stage w // G, partition rank w % G (the worker order of train_hybrid,
engines_impl.hpp:564-566). Stage groups link with gp_link_group_ipc (halo rows pulled
from peers' buffers, rank-ordered weight-gradient fold); adjacent stages of the same
rank link with gp_link_ipc. gloo is only the control plane (blob exchange). All
workers may share one GPU. Rank 0 writes the loss sums and every layer's parameters.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2308_10087_b200 as gp  # noqa: E402
from paper_2308_10087_b200 import distributed as D  # noqa: E402

ER500 = (500, 0.02, 3, 16, 5, 9)


def dataset(case):
    if case.get("data") == "powerlaw":  # tests/golden/powerlaw_2k (Chung-Lu, max degree 822)
        return gp.Dataset.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "powerlaw_2k"))
    return gp.Dataset.synthetic_er(*ER500)


def main():
    out, case = sys.argv[1], json.loads(sys.argv[2])
    kind, L, H, S, G, K = case["kind"], case["L"], case["H"], case["S"], case["G"], case["K"]
    epochs, seed = case["epochs"], case["seed"]
    import torch.distributed as dist
    dist.init_process_group("gloo")
    w, W = dist.get_rank(), dist.get_world_size()
    assert W == S * G
    s, r = w // G, w % G
    ds = dataset(case)
    part, _, _ = gp.partition_vertices(ds, G, case["ps"])
    chunk_of = gp.make_chunks(ds, K, case["cs"])
    model = gp.ModelConfig(kind=kind, layers=L, hidden=H)
    specs = gp.build_layer_specs(model, ds.num_features, ds.num_classes)
    params = gp.init_params(model, ds.num_features, ds.num_classes, seed)
    lo, hi = gp.make_stage_assignment(L, S)[s]
    eng = gp.StageEngine(num_vertices=ds.num_vertices, num_chunks=K, specs=specs, stage=s, num_stages=S,
                         layer_range=(lo, hi), hidden=H, num_classes=ds.num_classes, dropout=model.dropout,
                         seed=seed, fix_alpha=case.get("fix_alpha", 10),
                         historical_gradients=case.get("hist", False), synchronous_mode=case.get("sync", False),
                         device=w % max(1, gp.device_count()), group_size=G, group_rank=r)
    if G > 1:
        eng.upload_partition(part)
    off, cols, vals = ds.normalize_adjacency(model.self_loops)
    eng.upload_graph(off, cols, vals, chunk_of)
    x, lab, sp = ds.arrays()
    if s == 0:
        eng.upload_features(x)
    if s == S - 1:
        eng.upload_labels(lab, sp)
    for l in range(lo, hi):
        eng.set_params(l, *params[l])
    # stage links: same partition rank, adjacent stages
    up, down = eng.ipc_export() if S > 1 else (None, None)
    allb = [None] * W
    dist.all_gather_object(allb, (s, r, up, down))
    up_peer = next((d for (s2, r2, _, d) in allb if s2 == s - 1 and r2 == r), None)
    down_peer = next((u for (s2, r2, u, _) in allb if s2 == s + 1 and r2 == r), None)
    if S > 1:
        eng.link_ipc(up_peer, down_peer)
    if G > 1:
        eng.link_group_ipc(D.exchange_group_blobs(dist, s, r, G, eng.group_export()))
    losses = []
    for t in range(1, epochs + 1):
        st = eng.run_epoch(t, gp.shuffle_chunk_order(K, t, seed))
        if st.has_quality:
            losses.append(st.loss_sum)
    mine = {"s": s, "r": r, "losses": losses, "params": {l: eng.get_params(l) for l in range(lo, hi)}}
    eng.close()
    allr = [None] * W
    dist.all_gather_object(allr, mine)
    if w == 0:
        last = [m for m in allr if m["s"] == S - 1]
        last.sort(key=lambda m: m["r"])
        loss = np.zeros(epochs)
        for m in last:  # reduce_metrics: rank order (engines_impl.hpp:131-151)
            loss = loss + np.array(m["losses"], np.float64)
        arrs = {"loss_sum": loss}
        for m in allr:
            if m["r"] != 0:
                continue  # params come from each group's rank 0 (engines_impl.hpp:901-905)
            for l, (Wt, b) in m["params"].items():
                arrs[f"W{l}"], arrs[f"b{l}"] = Wt, b
        np.savez(out, **arrs)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
