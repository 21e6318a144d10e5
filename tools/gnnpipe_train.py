#!/usr/bin/env python3
"""Train on the B200 engine and write the run outputs of the reference's `gnnsim train`
(proj/tools/gnnsim.cpp:242-276): metrics.csv, trace.jsonl, comm_report.csv and one stage_<s>.ckpt
per pipeline stage, plus state.ckpt (parameters + Adam moments, for --resume).

    python tools/gnnpipe_train.py --synthetic er:4096:0.0039:1:128:16:1 --model gcnii --layers 8 \\
        --hidden 64 --stages 2 --chunks 8 --epochs 20 --out runs/er4k
    python tools/gnnpipe_train.py --dataset DIR ...          # a save_dataset directory
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2308_10087_b200 as gp  # noqa: E402

KINDS = {"gcn": gp.ModelKind.GCN, "sage": gp.ModelKind.SAGE, "gcnii": gp.ModelKind.GCNII}


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--dataset", help="dataset directory (load_dataset)")
    src.add_argument("--synthetic", help="er:N:P:GRAPH_SEED:F:C:FEATURE_SEED")
    ap.add_argument("--model", choices=sorted(KINDS), default="gcnii")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--hidden", type=int, default=64)
    ap.add_argument("--stages", type=int, default=1)
    ap.add_argument("--parts", type=int, default=1, help="graph partitions per stage (hybrid when > 1)")
    ap.add_argument("--chunks", type=int, default=0, help="default 4 x stages (gnnsim.cpp:226)")
    ap.add_argument("--epochs", type=int, default=10)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--fix-alpha", type=int, default=10)
    ap.add_argument("--sync", action="store_true")
    ap.add_argument("--trace", action="store_true", help="collect the measured trace (chunks run serially)")
    ap.add_argument("--resume", default="", help="state.ckpt of an earlier run")
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)

    if a.dataset:
        ds = gp.Dataset.load(a.dataset)
    else:
        _, n, p, gs, f, c, fs = a.synthetic.split(":")
        ds = gp.Dataset.synthetic_er(int(n), float(p), int(gs), int(f), int(c), int(fs))
    K = a.chunks or 4 * a.stages
    chunk_of = gp.make_chunks(ds, K, a.seed)
    model = gp.ModelConfig(kind=KINDS[a.model], layers=a.layers, hidden=a.hidden)
    os.makedirs(a.out, exist_ok=True)
    opt = gp.TrainOptions(model=model, epochs=a.epochs, seed=a.seed, fix_alpha=a.fix_alpha,
                          synchronous_mode=a.sync, collect_trace=a.trace, resume_path=a.resume,
                          save_state_path=os.path.join(a.out, "state.ckpt"))
    if a.parts > 1:
        part, _, _ = gp.partition_vertices(ds, a.parts, a.seed)
        res = gp.train_hybrid(ds, part, chunk_of, a.stages, opt)
    else:
        res = gp.train_pipeline(ds, chunk_of, a.stages, opt)
    gp.write_run_outputs(res, a.out)
    for s, (lo, hi) in enumerate(gp.make_stage_assignment(len(res.params), a.stages)):
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
