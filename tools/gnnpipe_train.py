#!/usr/bin/env python3
"""Train on the B200 engine and write the run outputs of the reference's `gnnsim train`
(proj/tools/gnnsim.cpp:242-276): metrics.csv, trace.jsonl, comm_report.csv and one stage_<s>.ckpt
per pipeline stage, plus state.ckpt (parameters + Adam moments, for --resume). `--mode` picks the
trainer as `gnnsim train --mode` does (gnnsim.cpp:187-239, :284-302); `--compare` adds compare.csv
(measured vs analytic bytes per epoch, `gnnsim compare`, gnnsim.cpp:305-347).

    python tools/gnnpipe_train.py --synthetic er:4096:0.0039:1:128:16:1 --model gcnii --layers 8 \\
        --hidden 64 --stages 2 --chunks 8 --epochs 20 --out runs/er4k
    python tools/gnnpipe_train.py --dataset DIR ...          # a save_dataset directory
    python tools/gnnpipe_train.py --synthetic ... --mode graph --workers 4 --compare --out runs/g4
    python tools/gnnpipe_train.py ... --chunks-file runs/a/chunks.txt --parts-file runs/a/parts.txt ...

The chunk plan and partition a run used are written to OUT/chunks.txt and OUT/parts.txt (the
reference CLI's save_assignment format, partition.cpp:250-256).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2308_10087_b200 as gp  # noqa: E402

KINDS = {"gcn": gp.ModelKind.GCN, "sage": gp.ModelKind.SAGE, "gcnii": gp.ModelKind.GCNII}


def write_compare(path, mode, ds, model, res, stages, ways, alpha):
    """compare.csv rows of `gnnsim compare` (gnnsim.cpp:305-347): per epoch, the analytic bytes of the
    mode (graph: 2 alpha N sum of aggregating in_dims x 4; pipeline: volume_pipeline; hybrid: both)
    against the measured ledger."""
    specs = gp.build_layer_specs(model, ds.num_features, ds.num_classes)
    vecs = 2 if any(s.kind == gp.LayerKind.GCN2CONV for s in specs) else 1  # model_needs_h0
    n = ds.num_vertices
    halo = 2.0 * sum(alpha * n * s.in_dim * 4.0 for s in specs if s.aggregates)
    pipe = gp.comm_volumes(n, model.layers, model.hidden, stages, ways, alpha, vecs)["pipeline"]
    rows = []
    for e in range(res.metrics.shape[0]):
        g, p = int(res.comm[e, 0]), int(res.comm[e, 1])
        pred, meas = {"graph": (halo, g), "pipeline": (pipe, p), "hybrid": (halo + pipe, g + p)}.get(mode, (0.0, 0))
        rel = abs(pred - meas) / pred if pred > 0 else float(meas)
        rows.append(dict(mode=mode, n=n, layers=model.layers, hidden=model.hidden, stages=stages, ways=ways,
                         alpha=alpha, vecs=vecs, predicted_bytes=pred, measured_bytes=meas, rel_error=rel))
        print(f"epoch predicted={pred:.0f} measured={meas} rel_error={rel:.3g}")
    gp.write_compare_csv(path, rows)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--dataset", help="dataset directory (load_dataset)")
    src.add_argument("--synthetic", help="er:N:P:GRAPH_SEED:F:C:FEATURE_SEED")
    ap.add_argument("--model", choices=sorted(KINDS), default="gcnii")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--hidden", type=int, default=64)
    ap.add_argument("--mode", choices=("sequential", "graph", "pipeline", "hybrid"), default="")
    ap.add_argument("--stages", type=int, default=1)
    ap.add_argument("--workers", type=int, default=0, help="graph mode: partitions (default 2)")
    ap.add_argument("--parts", type=int, default=1, help="graph partitions per stage (hybrid when > 1)")
    ap.add_argument("--compare", action="store_true", help="write compare.csv (measured vs analytic bytes)")
    ap.add_argument("--chunks", type=int, default=0, help="default 4 x stages (gnnsim.cpp:226)")
    ap.add_argument("--epochs", type=int, default=10)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--fix-alpha", type=int, default=10)
    ap.add_argument("--sync", action="store_true")
    ap.add_argument("--trace", action="store_true", help="collect the measured trace (chunks run serially)")
    ap.add_argument("--resume", default="", help="state.ckpt of an earlier run")
    ap.add_argument("--chunks-file", default="",
                    help="chunks.txt to train with (load_assignment); the plan used is written to OUT/chunks.txt")
    ap.add_argument("--parts-file", default="", help="parts.txt (hybrid / graph mode partition); written to OUT")
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)

    if a.dataset:
        ds = gp.Dataset.load(a.dataset)
    else:
        _, n, p, gs, f, c, fs = a.synthetic.split(":")
        ds = gp.Dataset.synthetic_er(int(n), float(p), int(gs), int(f), int(c), int(fs))
    mode = a.mode or ("hybrid" if a.parts > 1 else "pipeline")
    K = a.chunks or 4 * a.stages
    model = gp.ModelConfig(kind=KINDS[a.model], layers=a.layers, hidden=a.hidden)
    os.makedirs(a.out, exist_ok=True)
    opt = gp.TrainOptions(model=model, epochs=a.epochs, seed=a.seed, fix_alpha=a.fix_alpha,
                          synchronous_mode=a.sync, collect_trace=a.trace, resume_path=a.resume,
                          save_state_path=os.path.join(a.out, "state.ckpt"))
    stages, ways, alpha = a.stages, 1, 0.0

    def chunk_plan():  # make_chunks, or a chunks.txt (partition.cpp:250-269); saved next to the outputs
        if a.chunks_file:
            k, co = gp.load_assignment(a.chunks_file)
            if co.size != ds.num_vertices:
                raise SystemExit(f"{a.chunks_file}: {co.size} vertices, dataset has {ds.num_vertices}")
        else:
            k, co = K, gp.make_chunks(ds, K, a.seed)
        gp.save_assignment(os.path.join(a.out, "chunks.txt"), k, co)
        return co

    def partition(parts):
        if a.parts_file:
            g, part = gp.load_assignment(a.parts_file)
            if part.size != ds.num_vertices:
                raise SystemExit(f"{a.parts_file}: {part.size} vertices, dataset has {ds.num_vertices}")
            # boundary total sum_i |B_i| (partition.cpp:28-50): vertices outside part i with a neighbour in it
            off, cols, _ = ds.normalize_adjacency(True)
            rows = np.repeat(np.arange(ds.num_vertices, dtype=np.int64), np.diff(off).astype(np.int64))
            cross = part[rows] != part[cols]
            bt = int(np.unique(rows[cross] * g + part[cols[cross]]).size)
        else:
            part, _, bt = gp.partition_vertices(ds, parts, a.seed)
            g = parts
        gp.save_assignment(os.path.join(a.out, "parts.txt"), g, part)
        return part, bt
    if mode == "sequential":
        stages = 1
        res = gp.train_sequential(ds, opt)
    elif mode == "graph":
        stages = 1  # compare.csv's ways column is the group size (1) in graph mode (gnnsim.cpp:314)
        part, bt = partition(a.workers or 2)
        alpha = bt / ds.num_vertices  # replication_factor (partition.cpp:200-204)
        res = gp.train_graph_parallel(ds, part, opt)
    elif mode == "hybrid":
        ways = a.parts
        part, bt = partition(ways)
        alpha = bt / ds.num_vertices
        res = gp.train_hybrid(ds, part, chunk_plan(), a.stages, opt)
    else:
        res = gp.train_pipeline(ds, chunk_plan(), a.stages, opt)
    if a.compare:
        write_compare(os.path.join(a.out, "compare.csv"), mode, ds, model, res, stages, ways, alpha)
    gp.write_run_outputs(res, a.out)
    for s, (lo, hi) in enumerate(gp.make_stage_assignment(len(res.params), stages)):
        gp.save_stage_checkpoint(os.path.join(a.out, f"stage_{s}.ckpt"), model, ds.num_features, ds.num_classes,
                                 res.params, lo, hi)
    for row in res.metrics:
        print(f"epoch {int(row[0]):3d} loss {row[1]:.6f} train {row[2]:.4f} val {row[3]:.4f} test {row[4]:.4f} "
              f"{row[5] * 1e3:.2f} ms")
    if a.trace and len(res.trace):
        b = gp.bubble_analysis(res.trace)
        print(f"bubble measured {b['measured_bubble']:.3f} ideal {b['ideal_bubble']:.3f}")


if __name__ == "__main__":
    main()
