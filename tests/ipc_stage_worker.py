"""One pipeline stage per process over the CUDA-IPC transport (gp_link_ipc).

Launched by tests/test_gpu_ipc.py as
    python -m torch.distributed.run --nproc-per-node S --master-addr 127.0.0.1 \
        --master-port P tests/ipc_stage_worker.py OUT.npz [EPOCHS]
Every rank drives one StageEngine (all ranks may share one GPU: IPC works between
processes on the same device, which is how the single-GPU box exercises the
one-process-per-GPU path). gloo is only the control plane (blob exchange). Rank 0
writes the per-epoch loss sums (from the last stage) and every layer's parameters.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2308_10087_b200 as gp  # noqa: E402
from paper_2308_10087_b200 import distributed as D  # noqa: E402

N, P_EDGE, F, CLASSES, H, LAYERS, K = 900, 14.0 / 900, 24, 5, 16, 8, 4


def problem():
    ds = gp.Dataset.synthetic_er(N, P_EDGE, 1, F, CLASSES, 1)
    model = gp.ModelConfig(kind=gp.ModelKind.GCNII, layers=LAYERS, hidden=H, dropout=0.5)
    chunk_of = gp.make_chunks(ds, K, 1)
    return ds, model, chunk_of


def stage_engine(ds, model, chunk_of, rank, S, device):
    off, cols, vals = ds.normalize_adjacency(True)
    x, lab, sp = ds.arrays()
    specs = gp.build_layer_specs(model, F, CLASSES)
    params = gp.init_params(model, F, CLASSES, 1)
    lo, hi = gp.make_stage_assignment(LAYERS, S)[rank]
    eng = gp.StageEngine(num_vertices=N, num_chunks=K, specs=specs, stage=rank, num_stages=S, layer_range=(lo, hi),
                         hidden=H, num_classes=CLASSES, dropout=0.5, seed=1, device=device)
    eng.upload_graph(off, cols, vals, chunk_of)
    if rank == 0:
        eng.upload_features(x)
    if rank == S - 1:
        eng.upload_labels(lab, sp)
    for l in range(lo, hi):
        eng.set_params(l, *params[l])
    return eng, (lo, hi)


def main():
    out = sys.argv[1]
    epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    import torch.distributed as dist
    dist.init_process_group("gloo")
    rank, S = dist.get_rank(), dist.get_world_size()
    ds, model, chunk_of = problem()
    eng, (lo, hi) = stage_engine(ds, model, chunk_of, rank, S, rank % max(1, gp.device_count()))
    eng.link_ipc(*D.exchange_ipc_blobs(dist, rank, S, eng.ipc_export()))
    losses = []
    for t in range(1, epochs + 1):
        st = eng.run_epoch(t, gp.shuffle_chunk_order(K, t, 1))
        if st.has_quality:
            losses.append(st.loss_sum)
    mine = {"losses": losses, "params": {l: eng.get_params(l) for l in range(lo, hi)}}
    eng.close()
    allr = [None] * S
    dist.all_gather_object(allr, mine)
    if rank == 0:
        arrs = {"losses": np.array(allr[S - 1]["losses"], np.float64)}
        for r in allr:
            for l, (W, b) in r["params"].items():
                arrs[f"W{l}"], arrs[f"b{l}"] = W, b
        np.savez(out, **arrs)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
