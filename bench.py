#!/usr/bin/env python3
"""Headline benchmark: per-epoch time of chunk-pipelined 64-layer GCNII training on a
Reddit-shaped synthetic graph (BASELINE.json configs[2]), 1 stage per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank = one pipeline stage)

A step is one training epoch (forward + backward over all K chunks, parameter gradients,
Adam) over the whole graph, with the graph, features and stashes resident in HBM.
Timing: barrier + device sync on both sides, CUDA events on each stage's compute
stream, max over ranks. Rank 0 prints ONE JSON line.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (N, directed entries 2E, F, C, H, model, layers, description)
    "reddit": (232965, 114615892, 602, 41, 100, "gcnii", 64,
               "Reddit-shaped ER graph (232,965 vertices, 114.6M directed edges, 602 feat, 41 classes), "
               "64-layer GCNII H=100, historical embeddings"),
    "arxiv": (169343, 2332486, 128, 40, 128, "gcn", 16,
              "ogbn-arxiv-shaped ER graph (169,343 vertices, 2.33M directed edges, 128 feat, 40 classes), 16-layer GCN"),
    "er4k": (4096, 65520, 128, 16, 128, "gcn", 8,
             "ER 4K vertices avg-deg 16, 128 feat, 16 classes, 8-layer GCN"),
    # 64 layers need ~560 GB of stashes at S=1 (70 GB per stage at S=8); on one GPU use --layers 8,
    # the work of one of the 8 stages
    "products": (2449029, 123718280, 100, 47, 128, "gcnii", 64,
                 "ogbn-products-shaped ER graph (2,449,029 vertices, 123.7M directed edges, 100 feat, 47 classes), "
                 "GCNII H=128"),
}
METRIC = "epoch time, 64-layer GCNII full-graph, 1/2/4/8 B200; SpMM GB/s vs HBM peak"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- reference arm
def reference_epoch(args, S, K, steps):
    """Times the reference's own CPU kernels (oracle/_ref) on a bounded row sample and
    assembles the epoch time of an S-stage pipeline: max stage work x (K+S-1)/K."""
    from oracle.blob import REF_DRIVER, read_blob
    if not os.path.exists(REF_DRIVER):
        return None, "oracle/_ref/ref_driver not built"
    N, E2, F, Cc, H, model, L, _ = WORKLOADS[args.workload]
    L = args.layers or L
    p = E2 / (N * (N - 1))
    threads = 1  # per-row cost of one reference worker; stages run as parallel threads
    rows = args.ref_rows
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "b.blob")
        cmd = [REF_DRIVER, "bench", f"spec=er:{N}:{p!r}:1:{F}:{Cc}:1", f"model={model}", f"layers={L}",
               f"hidden={H}", f"rows={rows}", f"steps={steps}", f"threads={threads}", f"out={out}"]
        t0 = time.perf_counter()
        r = subprocess.run(cmd, capture_output=True, text=True)
        wall = time.perf_counter() - t0
        if r.returncode != 0:
            return None, f"ref_driver bench failed: {r.stderr.strip()[:200]}"
        d = read_blob(out)
    per = d["layer_epoch_seconds"].reshape(steps, L)
    import paper_2308_10087_b200 as gp
    ranges = gp.make_stage_assignment(L, S)
    epochs = []
    for s in range(steps):
        stage_work = [float(per[s, lo:hi].sum()) for lo, hi in ranges]
        # each stage is one reference worker thread (fabric.cpp:401-422); GPipe fill/drain
        epochs.append(max(stage_work) * (K + S - 1) / K)
    sample = (f"{int(d['rows_sampled'][0])} evenly strided rows per layer kind (first/middle/last) "
              f"x {steps} steps of the reference per-row kernels + DropMask::make, extrapolated to "
              f"N={N} rows x {L} layers, S={S} stage threads, (K+S-1)/K fill/drain; sampler wall {wall:.1f}s")
    return {"epochs": epochs, "threads": min(S, os.cpu_count() or 1), "sample": sample}, None


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    S = world
    K = args.chunks or 4 * S
    res, err = reference_epoch(args, S, K, args.warmup + args.steps)
    N, E2, F, Cc, H, model, L, desc = WORKLOADS[args.workload]
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": err}))
        return
    ep = res["epochs"][args.warmup:]
    v = statistics.median(ep)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s/epoch", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": desc, "stages": S, "chunks": K, "layers": args.layers or L},
        "cpu_baseline": {"value": v, "unit": "s/epoch", "cores": res["threads"], "kind": "reference",
                         "sample": res["sample"]},
        "e2e": {"value": v, "unit": "s/epoch", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ----------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="reddit", choices=sorted(WORKLOADS))
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--chunks", type=int, default=0, help="K (default 4*S, gnnsim.cpp:226)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=600)
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="stage boundary transport for N>1: CUDA-IPC copy-engine rings (default) or NCCL send/recv")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        return

    import paper_2308_10087_b200 as gp

    # one rank per GPU; more ranks than GPUs share devices round-robin (a
    # functional check of the multi-process path on a 1-GPU box, not a timing)
    ndev = gp.device_count()
    dev = local % ndev if ndev else local
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")  # control plane only; stage data moves over gp_link_ipc / gp_link_nccl

    def barrier():
        if dist:
            dist.barrier()

    from paper_2308_10087_b200 import distributed as D

    def max_over_ranks(x):
        return D.max_over_ranks(dist, x)

    S = world
    K = args.chunks or 4 * S
    N, E2, F, Cc, H, mk, L, desc = WORKLOADS[args.workload]
    L = args.layers or L
    kind = {"gcn": gp.ModelKind.GCN, "gcnii": gp.ModelKind.GCNII}[mk]
    model = gp.ModelConfig(kind=kind, layers=L, hidden=H, dropout=0.5)
    p = E2 / (N * (N - 1))
    t0 = time.perf_counter()
    ds = gp.Dataset.synthetic_er(N, p, 1, F, Cc, 1)
    chunk_of = gp.make_chunks(ds, K, 1) if K > 1 else np.zeros(N, np.uint32)
    off, cols, vals = ds.normalize_adjacency(True)
    x, lab, sp = ds.arrays()
    specs = gp.build_layer_specs(model, F, Cc)
    params = gp.init_params(model, F, Cc, 1)
    ranges = gp.make_stage_assignment(L, S)
    lo, hi = ranges[rank]
    prep_s = time.perf_counter() - t0

    def make_engine():
        eng = gp.StageEngine(num_vertices=N, num_chunks=K, specs=specs, stage=rank, num_stages=S,
                             layer_range=(lo, hi), hidden=H, num_classes=Cc, dropout=0.5, seed=1, device=dev)
        return eng

    def upload(eng):
        eng.upload_graph(off, cols, vals, chunk_of)
        if rank == 0:
            eng.upload_features(x)
        if rank == S - 1:
            eng.upload_labels(lab, sp)
        for l in range(lo, hi):
            eng.set_params(l, *params[l])

    def link(eng):
        if S == 1:
            return
        if args.transport == "ipc":
            eng.link_ipc(*D.exchange_ipc_blobs(dist, rank, S, eng.ipc_export()))
        else:
            ids = D.exchange_unique_ids(dist, rank, S, gp.nccl_unique_id)
            eng.link_nccl(*D.boundary_ids(ids, rank, S))

    def order(t):
        return gp.shuffle_chunk_order(K, t, 1)

    eng = make_engine()
    upload(eng)
    link(eng)
    t = 0
    for _ in range(args.warmup):
        t += 1
        eng.run_epoch(t, order(t))
    eng.synchronize()
    barrier()
    launches = 0
    with ClockSampler(dev) as clk:
        eng.mark(0)
        losses = []
        for _ in range(args.steps):
            t += 1
            st = eng.run_epoch(t, order(t))
            launches += st.kernel_launches
            if st.has_quality:
                losses.append(st.loss_sum)
        eng.mark(1)
        ms = eng.elapsed_ms(0, 1)
    barrier()
    ms = max_over_ranks(ms)
    if dist:  # whole-job kernel count
        import torch
        lt = torch.tensor([float(launches)], dtype=torch.float64)
        dist.all_reduce(lt)
        launches = int(lt.item())
    if dist:  # the loss lives on the last stage
        box = [losses]
        dist.broadcast_object_list(box, src=S - 1)
        losses = box[0]
    ms_step = ms / args.steps

    # per-kernel device times from one extra, untimed profiling epoch
    eng.set_profiling(True)
    eng.reset_profile()
    t += 1
    eng.run_epoch(t, order(t))
    prof = eng.profile()
    eng.set_profiling(False)
    dev_bytes = eng.device_bytes()
    eng.close()
    del eng

    # end-to-end through the public API: host buffers in, parameters/metrics out
    e2e = None
    if not args.no_e2e:
        if S == 1:
            barrier()
            opt = gp.TrainOptions(model=model, epochs=args.steps, seed=1, device=dev)
            t0 = time.perf_counter()
            res = gp.train_pipeline(ds, chunk_of, 1, opt)
            e2e_s = time.perf_counter() - t0
            h2d = (off.nbytes + cols.nbytes + vals.nbytes + chunk_of.nbytes + x.nbytes + lab.nbytes + sp.nbytes +
                   sum(w.nbytes + b.nbytes for w, b in params))
            d2h = sum(w.nbytes + b.nbytes for w, b in res.params) + res.metrics.nbytes
        else:
            e = make_engine()
            barrier()
            t0 = time.perf_counter()
            upload(e)
            link(e)
            for tt in range(1, args.steps + 1):
                e.run_epoch(tt, order(tt))
            pr = [e.get_params(l) for l in range(lo, hi)]
            e2e_s = max_over_ranks(time.perf_counter() - t0)
            h2d = off.nbytes + cols.nbytes + vals.nbytes + chunk_of.nbytes + (x.nbytes if rank == 0 else 0)
            d2h = sum(w.nbytes + b.nbytes for w, b in pr)
            e.close()
        e2e = {"value": e2e_s / args.steps, "unit": "s/epoch", "h2d_bytes_per_step": int(h2d // args.steps),
               "d2h_bytes_per_step": int(d2h // args.steps),
               "note": "public-API call train_pipeline(epochs=steps) incl. host CSR normalisation, H2D of the "
                       "graph/features/labels, all epochs and D2H of parameters+metrics, divided by steps"}

    cpu = None
    if rank == 0 and S == 1 and not args.no_cpu_baseline:
        res, err = reference_epoch(args, 1, K, 2)
        if res is None:
            cpu = {"value": None, "unavailable": err}
        else:
            cpu = {"value": statistics.median(res["epochs"]), "unit": "s/epoch", "cores": res["threads"],
                   "kind": "reference", "sample": res["sample"]}

    if rank != 0:
        return
    hbm, src = peaks()
    fa = prof["fwd_agg"]
    achieved = fa["alg_bytes"] / (fa["ms"] / 1e3) / 1e9 if fa["ms"] > 0 else None
    gather_rate = fa["gather_bytes"] / (fa["ms"] / 1e3) / 1e9 if fa["ms"] > 0 else None
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tp):
        try:
            t = json.load(open(tp)).get(args.workload)
            if t and L == WORKLOADS[args.workload][6]:
                # ncu DRAM bytes per row x the average rows of one launch (one chunk), in bytes
                traffic = t["dram_bytes_per_row"] * N / K
                traffic_src = t["source"]
        except Exception:
            traffic = None
    alg_per_launch = fa["alg_bytes"] / fa["launches"] if fa["launches"] else None
    agg_layers = sum(1 for s in specs if s.aggregates)
    edges_per_s = 2.0 * (E2) * agg_layers * 2 / (ms_step / 1e3)
    total_ms = sum(v["ms"] for v in prof.values())
    line = {
        "metric": METRIC, "value": ms_step / 1e3, "unit": "s/epoch", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (generate_er graph + hashed features, seed 1)",
        "config": {"workload": desc, "num_vertices": N, "nnz_norm_adj": int(cols.size), "features": F,
                   "classes": Cc, "hidden": H, "layers": L, "model": mk, "stages": S, "chunks": K,
                   "parallelism": f"pp{S}", "transport": args.transport if S > 1 else None,
                   "ranks_per_gpu": -(-world // max(1, ndev)), "l2_policy": f"inputs larger than L2 (stage stash {dev_bytes/2**30:.1f} GiB)"},
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": int(launches),
        "edges_per_s": edges_per_s,
        "roofline": {"kernel": "k_fwd8<FWD_GCN2, split> (CSR SpMM gather + GCNII initial-residual mix -> pre; the transform runs in k_fwd_tile)",
                     "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": (achieved / hbm) if achieved else None, "peak_source": src,
                     # DRAM read + write bytes per launch (ncu) next to the algorithmic bytes per launch
                     "traffic": traffic, "traffic_unit": "bytes/launch", "traffic_source": traffic_src,
                     "alg_bytes_per_launch": alg_per_launch,
                     "l2_gather_gbs": gather_rate,
                     # the binding roof of the gather: random 416-byte rows from the
                     # L2-resident table through LDG.256, measured by tools/tex_gather_bench.cu
                     "gather_ceiling_gbs": 16374.0,
                     "gather_frac": (gather_rate / 16374.0) if gather_rate else None,
                     "share_of_step": fa["ms"] / total_ms if total_ms else None},
        "cpu_baseline": cpu,
        "kernel_ms_per_epoch": {k: round(v["ms"], 3) for k, v in prof.items() if v["launches"]},
        "host_prep_s": round(prep_s, 2),
        "loss_last": (losses[-1] / float((sp == 1).sum())) if losses else None,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
