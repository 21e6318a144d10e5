"""Generate the golden fixtures in tests/golden/ from the reference itself.

Runs oracle/_ref/ref_driver (the unmodified gnnsim sources compiled by oracle/Makefile) and
stores its outputs as small .npz files. Re-run after changing a scenario:

    make -C oracle && python tests/golden/make_golden.py
"""
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.blob import run_ref  # noqa: E402

# Dataset spec strings are passed verbatim to both the reference and the product.
ER500 = "er:500:0.02:3:16:5:9"
ER300W = "er:300:0.03:11:40:7:2"  # F=40 > nothing special; used for GCN first layer width != H

# BASELINE.json configs at their own shapes (bench.py WORKLOADS; p = directed entries / (N (N-1)))
CFG0 = "er:4096:" + repr(65536 / (4096 * 4095)) + ":1:128:16:1"
CFG1 = "er:169343:" + repr(2332486 / (169343 * 169342)) + ":1:128:40:1"
CFG2 = "er:232965:" + repr(114615892 / (232965 * 232964)) + ":1:602:41:1"
BIG = {  # full-size scenarios: chunk_of is stored as its sha256, the forward dump is compact
    # configs[0] exactly: ER-4K, F=H=128, C=16, 8-layer GCN, K=4, S=1, 20 epochs
    "cfg0_er4k_gcn8_s1k4_20ep": ("train", dict(spec=CFG0, model="gcn", layers=8, hidden=128, S=1, K=4, chunk_seed=1,
                                               epochs=20, seed=1)),
    # configs[1] at the real ogbn-arxiv shape: 16-layer GCN, 2 stages x 8 chunks and 4 x 16
    "cfg1_arxiv_gcn16_s2k8_3ep": ("train", dict(spec=CFG1, model="gcn", layers=16, hidden=128, S=2, K=8,
                                                chunk_seed=1, epochs=3, seed=1, fabric="conc")),
    "cfg1_arxiv_gcn16_s4k16_3ep": ("train", dict(spec=CFG1, model="gcn", layers=16, hidden=128, S=4, K=16,
                                                 chunk_seed=1, epochs=3, seed=1, fabric="conc")),
    # configs[2] at the full Reddit shape with 4 layers (Dense 602->100, 2 Gcn2Conv, Dense 100->41):
    # whole-graph epoch-1 loss and every parameter gradient; 2 pipeline epochs at K=4 (params after Adam)
    "cfg2_reddit_gcnii4_forward": ("forward", dict(spec=CFG2, model="gcnii", layers=4, hidden=100, seed=1, epoch=1,
                                                   full=0)),
    "cfg2_reddit_gcnii4_s1k4_2ep": ("train", dict(spec=CFG2, model="gcnii", layers=4, hidden=100, S=1, K=4,
                                                  chunk_seed=1, epochs=2, seed=1)),
    # configs[2] itself: the headline 64-layer GCNII at the Reddit shape, 8 stages x 32 chunks (the
    # reference runs one worker thread per stage), 2 epochs
    "cfg2_reddit_gcnii64_s8k32_2ep": ("train", dict(spec=CFG2, model="gcnii", layers=64, hidden=100, S=8, K=32,
                                                    chunk_seed=1, epochs=2, seed=1, fabric="conc", watchdog=36000)),
    # configs[1] over the north star's 20-epoch loss-curve horizon at the real arxiv shape
    "cfg1_arxiv_gcn16_s2k8_20ep": ("train", dict(spec=CFG1, model="gcn", layers=16, hidden=128, S=2, K=8,
                                                 chunk_seed=1, epochs=20, seed=1, fabric="conc", watchdog=36000)),
}

SCENARIOS = {
    # name: (cmd, kwargs)
    "graph_er500": ("graph", dict(spec=ER500)),
    "graph_g8": ("graph", dict(spec="g8:2:2")),
    "chunks_er500_k1": ("chunks", dict(spec=ER500, K=1, seed=5)),
    "chunks_er500_k4": ("chunks", dict(spec=ER500, K=4, seed=5)),
    "chunks_er500_k7": ("chunks", dict(spec=ER500, K=7, seed=5)),
    "graph_sbm4x100": ("graph", dict(spec="sbm:4:100:0.2:0.002:31")),
    "chunks_sbm4x100_k4": ("chunks", dict(spec="sbm:4:100:0.2:0.002:31", K=4, seed=31)),
    "shuffle_k8": ("shuffle", dict(K=8, seed=3, epochs=20)),
    "forward_gcn": ("forward", dict(spec=ER500, model="gcn", layers=3, hidden=16, seed=7, epoch=1)),
    "forward_gcnii": ("forward", dict(spec=ER500, model="gcnii", layers=5, hidden=16, seed=7, epoch=1)),
    "forward_sage": ("forward", dict(spec=ER500, model="sage", layers=3, hidden=16, seed=7, epoch=1)),
    "train_sage_s2k4": ("train", dict(spec=ER500, model="sage", layers=4, hidden=16, S=2, K=4, chunk_seed=3,
                                      epochs=10, seed=46, fix_alpha=3)),
    "forward_sage_wide": ("forward", dict(spec="er:300:0.03:11:200:7:2", model="sage", layers=3, hidden=16, seed=7,
                                          epoch=1)),
    "train_sage_wide_s2k4": ("train", dict(spec="er:300:0.03:11:200:7:2", model="sage", layers=3, hidden=16, S=2, K=4,
                                           chunk_seed=1, epochs=6, seed=50, fix_alpha=2)),
    # BASELINE configs[1] in miniature, 20-epoch loss curve: arxiv-like density (avg degree ~14),
    # 16-layer GCN, 2 stages, 8 chunks, default staleness (fix_alpha 10)
    "train_gcn16_arxivlike_s2k8_20ep": ("train", dict(spec="er:20000:0.0007:21:128:40:5", model="gcn", layers=16,
                                                      hidden=64, S=2, K=8, chunk_seed=6, epochs=20, seed=61,
                                                      fix_alpha=10)),
    # BASELINE configs[4] in miniature: hybrid pipeline x graph parallel GCNII on a power-law graph
    # (tests/golden/powerlaw_2k, make_powerlaw.py; hubs of degree 822 next to degree-1 leaves)
    "train_gcnii_powerlaw_hyb_s2g2": ("train", dict(spec="dir:" + os.path.join(HERE, "powerlaw_2k"), model="gcnii",
                                                    layers=8, hidden=16, S=2, G=2, K=4, chunk_seed=3, part_seed=1,
                                                    epochs=8, seed=51, fix_alpha=3)),
    "train_gcn_powerlaw_s2k8": ("train", dict(spec="dir:" + os.path.join(HERE, "powerlaw_2k"), model="gcn", layers=4,
                                              hidden=16, S=2, K=8, chunk_seed=4, epochs=8, seed=52, fix_alpha=2)),
    "train_sage_hyb_s2g2": ("train", dict(spec=ER500, model="sage", layers=4, hidden=16, S=2, G=2, K=4, chunk_seed=3,
                                          part_seed=1, epochs=8, seed=48, fix_alpha=3)),
    "train_sage_hyb_s1g2_hist": ("train", dict(spec=ER500, model="sage", layers=3, hidden=12, S=1, G=2, K=4,
                                               chunk_seed=5, part_seed=2, epochs=6, seed=49, fix_alpha=2, hist=1)),
    "train_sage_s1k4_hist": ("train", dict(spec=ER500, model="sage", layers=3, hidden=16, S=1, K=4, chunk_seed=3,
                                           epochs=8, seed=47, fix_alpha=2, hist=1)),
    "train_gcn_s1k1": ("train", dict(spec=ER500, model="gcn", layers=4, hidden=16, S=1, K=1, epochs=10, seed=42)),
    "train_gcn_s2k4": ("train", dict(spec=ER500, model="gcn", layers=4, hidden=16, S=2, K=4, chunk_seed=3,
                                     epochs=10, seed=42, fix_alpha=3)),
    "train_gcnii_s2k4": ("train", dict(spec=ER500, model="gcnii", layers=6, hidden=16, S=2, K=4, chunk_seed=3,
                                       epochs=10, seed=43, fix_alpha=3)),
    "train_gcnii_s1k4_sync": ("train", dict(spec=ER500, model="gcnii", layers=6, hidden=16, S=1, K=4,
                                            chunk_seed=3, epochs=10, seed=44, sync=1)),
    "train_gcn_hyb_s2g2": ("train", dict(spec=ER500, model="gcn", layers=4, hidden=16, S=2, G=2, K=4, chunk_seed=3,
                                         part_seed=1, epochs=8, seed=42, fix_alpha=3)),
    "train_gcnii_hyb_s2g2": ("train", dict(spec=ER500, model="gcnii", layers=6, hidden=16, S=2, G=2, K=4,
                                           chunk_seed=3, part_seed=2, epochs=8, seed=43, fix_alpha=3)),
    "train_gcnii_hyb_s1g3_sync": ("train", dict(spec=ER500, model="gcnii", layers=5, hidden=16, S=1, G=3, K=3,
                                                chunk_seed=5, part_seed=3, epochs=6, seed=44, sync=1)),
    "train_gcn_hyb_s3g2_hist": ("train", dict(spec=ER500, model="gcn", layers=6, hidden=12, S=3, G=2, K=6,
                                              chunk_seed=7, part_seed=4, epochs=6, seed=45, fix_alpha=2, hist=1)),
    "train_gcn_graph_p3": ("train", dict(spec=ER500, model="gcn", layers=3, hidden=16, mode="graph", G=3,
                                         part_seed=5, epochs=6, seed=53)),
    "train_gcnii_graph_p2": ("train", dict(spec=ER500, model="gcnii", layers=5, hidden=16, mode="graph", G=2,
                                           part_seed=6, epochs=6, seed=54)),
    "train_gcn_s3k6_w40": ("train", dict(spec=ER300W, model="gcn", layers=6, hidden=24, S=3, K=6, chunk_seed=1,
                                         epochs=8, seed=45, fix_alpha=2)),
}


def analytics_events():
    """A deterministic 3-worker, 5-chunk trace with every event kind (input of the analytics golden)."""
    rng = np.random.default_rng(2308)
    rows = []
    for w in range(3):
        t = 0.01 * w
        for k in range(5):
            if w:
                idle = float(rng.uniform(0, 0.004))
                rows.append((w, 3, k, 2 * w, 2 * w + 1, t, t + idle))
                t += idle
                rows.append((w, 2, k, 2 * w, 2 * w + 1, t, t))
            dt = float(rng.uniform(0.005, 0.02))
            rows.append((w, 0, k, 2 * w, 2 * w + 1, t, t + dt))
            t += dt
            if w < 2:
                rows.append((w, 1, k, 2 * w, 2 * w + 1, t, t))
        rows.append((w, 0, -1, 2 * w, 2 * w + 1, t, t + 0.002))
    return rows


def golden_analytics(td):
    ev = analytics_events()
    path = os.path.join(td, "events.txt")
    with open(path, "w") as f:
        for r in ev:
            f.write(" ".join(repr(x) for x in r) + "\n")
    d = run_ref("analytics", os.path.join(td, "analytics.blob"), **{"in": path, "dir": td})
    files = {}
    for name in ("trace.jsonl", "comm_report.csv", "metrics.csv", "compare.csv"):
        with open(os.path.join(td, name)) as f:
            files["file_" + name.replace(".", "_")] = np.array(f.read())
    arr = np.array([(w, k, c, lo, hi, 0, t0, t1) for (w, k, c, lo, hi, t0, t1) in ev],
                   dtype=[("worker", np.uint32), ("kind", np.uint32), ("chunk", np.int32), ("layer_lo", np.int32),
                          ("layer_hi", np.int32), ("reserved", np.uint32), ("t_start", np.float64),
                          ("t_end", np.float64)])
    np.savez_compressed(os.path.join(HERE, "analytics.npz"), events=arr, **d, **files)
    print("analytics", sorted(d))


CKPTS = {
    # name: (model, layers, hidden, F, C, seed, lo, hi)
    "ckpt_gcnii": ("gcnii", 5, 6, 7, 3, 12, 0, 5),
    "ckpt_gcn_stage1": ("gcn", 4, 8, 10, 4, 3, 2, 4),
}


def golden_checkpoints(td):
    out = {}
    for name, (model, L, H, F, Cc, seed, lo, hi) in CKPTS.items():
        path = os.path.join(td, name + ".ckpt")
        run_ref("ckpt", os.path.join(td, name + ".blob"), model=model, layers=L, hidden=H, F=F, C=Cc, seed=seed,
                lo=lo, hi=hi, path=path)
        with open(path, "rb") as f:
            out[name] = np.frombuffer(f.read(), np.uint8)
        out[name + "_args"] = np.array([L, H, F, Cc, seed, lo, hi], np.int64)
    np.savez_compressed(os.path.join(HERE, "checkpoints.npz"), **out)
    print("checkpoints", sorted(out))


def make_big(name, td):
    import hashlib
    cmd, kw = BIG[name]
    d = run_ref(cmd, os.path.join(td, name + ".blob"), timeout=14400, **kw)
    if "chunk_of" in d:
        d["chunk_of_sha256"] = np.array(hashlib.sha256(d.pop("chunk_of").astype("<u4").tobytes()).hexdigest())
    meta = {"cmd": cmd, **{k: str(v) for k, v in kw.items()}}
    np.savez_compressed(os.path.join(HERE, name + ".npz"), __meta__=np.array(repr(meta)), **d)
    print(name, sorted(d)[:6], "...")


def golden_assignments(td):
    """chunks.txt / parts.txt written by the reference's save_assignment (partition.cpp:250-256)."""
    d = run_ref("assign", os.path.join(td, "assign.blob"), spec=ER500, K=4, seed=5, dir=td)
    files = {}
    for name in ("chunks.txt", "parts.txt"):
        with open(os.path.join(td, name)) as f:
            files["file_" + name.replace(".", "_")] = np.array(f.read())
    np.savez_compressed(os.path.join(HERE, "assign_er500_k4.npz"), **files, chunk_of=d["chunk_of"])
    print("assignments", sorted(files))


def main():
    names = sys.argv[1:]
    with tempfile.TemporaryDirectory() as td:
        if names:  # only the named scenarios (the full-size ones take minutes each on one core)
            for n in names:
                if n == "assignments":
                    golden_assignments(td)
                elif n in BIG:
                    make_big(n, td)
                else:
                    cmd, kw = SCENARIOS[n]
                    d = run_ref(cmd, os.path.join(td, n + ".blob"), **kw)
                    np.savez_compressed(os.path.join(HERE, n + ".npz"),
                                        __meta__=np.array(repr({"cmd": cmd, **{k: str(v) for k, v in kw.items()}})), **d)
            return
        golden_analytics(td)
        golden_checkpoints(td)
        golden_assignments(td)
        for name in BIG:
            make_big(name, td)
        for name, (cmd, kw) in SCENARIOS.items():
            d = run_ref(cmd, os.path.join(td, name + ".blob"), **kw)
            meta = {"cmd": cmd, **{k: str(v) for k, v in kw.items()}}
            np.savez_compressed(os.path.join(HERE, name + ".npz"), __meta__=np.array(repr(meta)), **d)
            print(name, sorted(d)[:6], "...")


if __name__ == "__main__":
    main()
