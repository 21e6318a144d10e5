"""Worker for tests/test_gpu_nccl.py: one pipeline stage linked through gp_link_nccl (test
infrastructure). Usage: nccl_stage_worker.py <stage> <id file> <out file>. Stage 0 writes a
fresh ncclUniqueId to <id file>; stage 1 reads it. Both processes sit on device 0 (the pool
has one GPU), which NCCL may refuse: the worker records the outcome instead of hanging."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2308_10087_b200 as gp  # noqa: E402


def main():
    stage, idf, outf = int(sys.argv[1]), sys.argv[2], sys.argv[3]
    ds = gp.Dataset.synthetic_er(500, 0.02, 3, 16, 5, 9)
    model = gp.ModelConfig(kind=gp.ModelKind.GCN, layers=4, hidden=16)
    specs = gp.build_layer_specs(model, ds.num_features, ds.num_classes)
    ranges = gp.make_stage_assignment(4, 2)
    co = gp.make_chunks(ds, 4, 3)
    eng = gp.StageEngine(num_vertices=ds.num_vertices, num_chunks=4, specs=specs, stage=stage, num_stages=2,
                         layer_range=ranges[stage], hidden=16, num_classes=ds.num_classes, dropout=0.5, seed=1)
    off, cols, vals = ds.normalize_adjacency(True)
    eng.upload_graph(off, cols, vals, co)
    x, lab, sp = ds.arrays()
    if stage == 0:
        eng.upload_features(x)
        uid = gp.nccl_unique_id()
        with open(idf + ".tmp", "wb") as f:
            f.write(uid)
        os.replace(idf + ".tmp", idf)
    else:
        eng.upload_labels(lab, sp)
        while not os.path.exists(idf):
            time.sleep(0.05)
        uid = open(idf, "rb").read()
    for l in range(*ranges[stage]):
        eng.set_params(l, *gp.init_params(model, ds.num_features, ds.num_classes, 1)[l])
    t0 = time.time()
    res = {"stage": stage}
    try:
        eng.link_nccl(uid if stage == 1 else None, uid if stage == 0 else None)
        res["linked"] = True
        losses = []
        for t in range(1, 4):
            st = eng.run_epoch(t, gp.shuffle_chunk_order(4, t, 1))
            if st.has_quality:
                losses.append(st.loss_sum)
        res["losses"] = losses
        res["params"] = [eng.get_params(l)[0].tolist() for l in range(*ranges[stage])]
    except gp.GnnsimError as e:
        res["error"] = f"{type(e).__name__}: {e}"
    res["seconds"] = time.time() - t0
    with open(outf, "w") as f:
        json.dump(res, f)


if __name__ == "__main__":
    main()
