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
    "er4k": (4096, 65536, 128, 16, 128, "gcn", 8,
             "ER 4K vertices avg-deg 16, 128 feat, 16 classes, 8-layer GCN"),
    # 64 layers need ~560 GB of stashes at S=1 (70 GB per stage at S=8); on one GPU use --layers 8,
    # the work of one of the 8 stages
    "products": (2449029, 123718280, 100, 47, 128, "gcnii", 64,
                 "ogbn-products-shaped ER graph (2,449,029 vertices, 123.7M directed edges, 100 feat, 47 classes), "
                 "GCNII H=128"),
}
METRIC = "epoch time, 64-layer GCNII full-graph, 1/2/4/8 B200; SpMM GB/s vs HBM peak"
DATA = "synthetic (generate_er graph + hashed features, seed 1)"


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


# ----------------------------------------------------------------------------- shared
def stage_ranges(L, S):
    """make_stage_assignment (engines.cpp:8-21) restated: near-equal consecutive layer
    split, the first L mod S stages get one extra. Kept here so the reference arm never
    imports the product package."""
    base, extra = divmod(L, S)
    out, lo = [], 0
    for s in range(S):
        hi = lo + base + (1 if s < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def workload_config(args, S, K):
    """The `config` object both arms print (identical keys and values)."""
    N, E2, F, Cc, H, mk, L, desc = WORKLOADS[args.workload]
    L = args.layers or L
    return {"workload": desc, "num_vertices": N, "directed_edges": E2, "features": F, "classes": Cc,
            "hidden": H, "layers": L, "model": mk, "stages": S, "chunks": K, "parallelism": f"pp{S}",
            "l2_policy": (f"inputs larger than L2: one epoch streams {L} layers of N x H fp32 stashes "
                          f"({N * H * 4 * L / 2**30:.1f} GiB per stash kind) through the 126 MB L2"
                          if N * H * 4 * L > 4 * 126e6 else
                          "inputs smaller than L2 (launch-bound shape; no flush between epochs)")}


# ----------------------------------------------------------------------------- reference arm
def reference_epochs(args, S, K):
    """Whole epochs of the reference's own train_pipeline<float> (engines_impl.hpp:911-920,
    oracle/_ref/ref_driver epochs; Fabric::Mode::Concurrent, one thread per stage worker)
    on the same synthetic graph and the same S stages, at two layer counts La and Lb = La + S
    (one more layer on every stage), run side by side: La = 3 at S = 1, else the smallest
    multiple of S that is >= 3. A 64-layer epoch on the host is hours, so the L-layer value is
    the projection t(La) + (L - La) * (t(Lb) - t(La)) / S, labelled as
    such."""
    from oracle.blob import REF_DRIVER, read_blob
    if not os.path.exists(REF_DRIVER):
        return None, "oracle/_ref/ref_driver not built"
    N, E2, F, Cc, H, model, L, _ = WORKLOADS[args.workload]
    L = args.layers or L
    p = E2 / (N * (N - 1))
    La = S * -(-max(3, S) // S)
    Lb = La + S
    Ls = (La, Lb) if L > 16 and L > Lb else (L,)  # up to 16 layers: the whole model is measured
    with tempfile.TemporaryDirectory() as td:
        procs = {}
        t0 = time.perf_counter()
        for l in Ls:
            out = os.path.join(td, f"e{l}.blob")
            cmd = [REF_DRIVER, "epochs", f"spec=er:{N}:{p!r}:1:{F}:{Cc}:1", f"model={model}", f"layers={l}",
                   f"hidden={H}", f"S={min(S, l)}", f"K={K}", "chunk_seed=1", "seed=1", "epochs=1", f"out={out}"]
            procs[l] = (subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True), out)
        res = {}
        for l, (pr, out) in procs.items():
            _, err = pr.communicate()
            if pr.returncode != 0:
                return None, f"ref_driver epochs failed: {err.strip()[:200]}"
            res[l] = read_blob(out)
        wall = time.perf_counter() - t0
    ep = {l: float(res[l]["epoch_s"][0]) for l in Ls}
    if len(Ls) == 2:
        marg = (ep[Lb] - ep[La]) / S
        full = ep[La] + (L - La) * marg
        how = (f"projection t({La})+(L-{La})*(t({Lb})-t({La}))/S from measured whole train_pipeline<float> epochs "
               f"at L={La} ({ep[La]:.1f} s) and L={Lb} ({ep[Lb]:.1f} s) over S={S} stages, marginal {marg:.1f} s "
               f"per layer")
    else:
        full = ep[L]
        how = f"measured whole train_pipeline<float> epoch at L={L} ({full:.2f} s)"
    g = res[Ls[0]]
    sample = (f"{how}; same graph/features/K/seed as the GPU arm, S={S} worker thread(s) per run, "
              f"runs side by side; excl. dataset gen ({float(g['gen_s'][0]):.1f} s), make_chunks "
              f"({float(g['chunk_s'][0]):.1f} s) and the call's setup ({float(g['setup_s'][0]):.1f} s); "
              f"CPU wall {wall:.0f} s")
    return {"value": full, "cores": S, "sample": sample, "projection": len(Ls) == 2,
            "measured_epoch_s": ep, "cpu_wall_s": wall, "cpu": cpu_info()}, None


def cpu_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    S = world
    K = args.chunks or 4 * S
    res, err = reference_epochs(args, S, K)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": err}))
        return
    v = res["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s/epoch", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": DATA,
        "config": workload_config(args, S, K),
        "cpu_baseline": {"value": v, "unit": "s/epoch", "cores": res["cores"], "kind": "reference",
                         "sample": res["sample"], "projection": res["projection"],
                         "measured_epoch_s": res["measured_epoch_s"], "cpu_wall_s": res["cpu_wall_s"],
                         "cpu": res["cpu"]},
        "e2e": {"value": v, "unit": "s/epoch", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("steps/warmup are not repeated on the CPU: one whole epoch per layer count is measured "
                 "(cpu_baseline.measured_epoch_s; the run's CPU wall is cpu_baseline.cpu_wall_s)"),
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
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="stage boundary transport for N>1: CUDA-IPC copy-engine rings (default) or NCCL send/recv")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: relaunch this script under torchrun with N ranks
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} disagrees with WORLD_SIZE={world}")
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
    # the dominant kernel (the forward SpMM gather) is timed live: CUDA events on its stream
    # around each of its launches inside the timed region (the wavefront stays on)
    eng.reset_profile()
    eng.set_live_timing("fwd_agg")
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
    live = eng.profile()["fwd_agg"]
    eng.set_live_timing(None)
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

    # occupied time per kernel class inside normal (wavefront) epochs: events around every
    # launch for two extra untimed epochs, reduced to the union of each class's launch intervals
    eng.reset_profile()
    eng.set_live_timing("all")
    for _ in range(2):
        t += 1
        eng.run_epoch(t, order(t))
    eng.synchronize()
    live_all = eng.profile()
    eng.set_live_timing(None)
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
            # train_pipeline ships the raw neighbour lists (u64 offsets, u32 neighbours); the
            # normalised, renumbered CSR is built on the device from them (k_build_edges)
            raw_graph = 8 * off.size + 4 * (cols.size - N)  # neighbours = normalised entries - self loops
            h2d = (raw_graph + chunk_of.nbytes + x.nbytes + lab.nbytes + sp.nbytes +
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
        res, err = reference_epochs(args, 1, K)
        if res is None:
            cpu = {"value": None, "unavailable": err}
        else:
            cpu = {"value": res["value"], "unit": "s/epoch", "cores": res["cores"], "kind": "reference",
                   "sample": res["sample"], "projection": res["projection"],
                   "measured_epoch_s": res["measured_epoch_s"], "cpu": res["cpu"]}

    if rank != 0:
        return
    hbm, src = peaks()
    fa = live  # timed region, wavefront on
    achieved = fa["alg_bytes"] / (fa["ms"] / 1e3) / 1e9 if fa["ms"] > 0 else None
    gather_rate = fa["gather_bytes"] / (fa["ms"] / 1e3) / 1e9 if fa["ms"] > 0 else None
    fs = prof["fwd_agg"]  # the serial profiling epoch (no concurrent kernels)
    achieved_serial = fs["alg_bytes"] / (fs["ms"] / 1e3) / 1e9 if fs["ms"] > 0 else None
    gather_serial = fs["gather_bytes"] / (fs["ms"] / 1e3) / 1e9 if fs["ms"] > 0 else None
    # the same bytes over the time the kernel occupied the GPU in the timed region (union of its
    # launch intervals: concurrent launches of two chunks on the wavefront streams count once)
    span = fa.get("span_ms", 0.0)
    achieved_span = fa["alg_bytes"] / (span / 1e3) / 1e9 if span > 0 else None
    gather_span = fa["gather_bytes"] / (span / 1e3) / 1e9 if span > 0 else None
    # DRAM bytes per launch of the dominant kernel from a committed `ncu --set full` capture
    # of the same build at this workload (tools/roofline_capture.py); K = 4 chunk launches
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tp):
        t = json.load(open(tp)).get(args.workload)
        if t and "dram_bytes_per_launch" in t:
            traffic = t["dram_bytes_per_launch"] * 4.0 / K
            traffic_src = t["source"]
    # the binding roof of the gather: uniformly random padded-row gathers from a table of
    # this workload's shape, measured by tools/gather_ceiling.cu (profiles/gather_ceiling.json)
    ceiling, ceiling_src = None, None
    cp = os.path.join(ROOT, "profiles", "gather_ceiling.json")
    if os.path.exists(cp):
        c = json.load(open(cp)).get(args.workload)
        if c:
            ceiling, ceiling_src = c.get("gbs"), c.get("source")
    alg_per_launch = fa["alg_bytes"] / fa["launches"] if fa["launches"] else None
    gathered = prof["fwd_agg"]["gather_bytes"] + prof["bwd_agg"]["gather_bytes"]  # one (profiling) epoch
    agg_layers = sum(1 for s in specs if s.aggregates)
    edges_per_s = 2.0 * (E2) * agg_layers * 2 / (ms_step / 1e3)
    total_ms = sum(v["ms"] for v in prof.values())
    line = {
        "metric": METRIC, "value": ms_step / 1e3, "unit": "s/epoch", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": DATA,
        "config": workload_config(args, S, K),
        "transport": args.transport if S > 1 else None, "ranks_per_gpu": -(-world // max(1, ndev)),
        "nnz_norm_adj": int(cols.size), "stage_stash_gib": round(dev_bytes / 2**30, 2),
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": int(launches),
        "edges_per_s": edges_per_s,
        "roofline": {"kernel": "k_fwd8<FWD_GCN|FWD_GCN2, 2, split> (CSR SpMM gather [+ GCNII initial-residual mix] -> pre; "
                               "the transform runs in k_tc_xform on tcgen05)",
                     # achieved: algorithmic bytes per launch / the kernel's effective launch duration
                     # in the timed region = its occupied time (union of the live launch intervals)
                     # / launches. Launches of different chunks overlap on the wavefront streams, so
                     # a single launch's own interval (achieved_live) counts the shared time twice.
                     "bound": "hbm", "achieved": achieved_span, "peak": hbm, "unit": "GB/s",
                     "frac": (achieved_span / hbm) if achieved_span else None, "peak_source": src,
                     # DRAM read + write bytes per launch (ncu) next to the algorithmic bytes per launch
                     "traffic": traffic, "traffic_unit": "bytes/launch", "traffic_source": traffic_src,
                     "alg_bytes_per_launch": alg_per_launch,
                     "l2_gather_gbs": gather_rate,
                     "gather_ceiling_gbs": ceiling, "gather_ceiling_source": ceiling_src,
                     "gather_frac": (gather_rate / ceiling) if gather_rate and ceiling else None,
                     # like for like with the ceiling microbenchmark (an isolated kernel): the serial epoch
                     "l2_gather_gbs_serial": gather_serial,
                     "gather_frac_serial": (gather_serial / ceiling) if gather_serial and ceiling else None,
                     "timing": (f"CUDA events around each of the {fa['launches']} launches of the kernel inside "
                                "the timed region (its stream; chunk wavefront on)"),
                     "ms_per_launch": span / fa["launches"] if fa["launches"] else None,
                     "ms_per_launch_live": fa["ms"] / fa["launches"] if fa["launches"] else None,
                     "achieved_live": achieved, "frac_live": (achieved / hbm) if achieved else None,
                     "achieved_serial": achieved_serial,
                     "span_share_of_step": (span / args.steps) / ms_step if ms_step else None,
                     "achieved_span": achieved_span,
                     "frac_span": (achieved_span / hbm) if achieved_span else None,
                     "l2_gather_gbs_span": gather_span,
                     "gather_frac_span": (gather_span / ceiling) if gather_span and ceiling else None,
                     "note": ("achieved (= achieved_span): algorithmic bytes over the time at least one "
                              "launch of the kernel was running (union of the live launch intervals, CUDA "
                              "events on each launch's stream), i.e. per launch over span / launches; "
                              "achieved_live: over each launch's own interval, which includes the launches "
                              "of other chunks co-running on the other wavefront streams (summed intervals = "
                              "share_of_step x the step); achieved_serial: over the isolated launch time of "
                              "the serial profiling epoch"),
                     "share_of_step": (fa["ms"] / args.steps) / ms_step if ms_step else None},
        # epoch-level bound: every byte the forward and backward SpMMs gather per epoch, at the
        # measured random-row gather ceiling of this shape, is a lower bound on the epoch time
        "epoch_gather_bound": ({
            "gathered_bytes": gathered, "ceiling_gbs": ceiling, "bound_s": gathered / (ceiling * 1e9),
            "frac": gathered / (ceiling * 1e9) / (ms_step / 1e3)} if ceiling else None),
        "cpu_baseline": cpu,
        "kernel_ms_per_epoch": {k: round(v["ms"], 3) for k, v in prof.items() if v["launches"]},
        # wavefront epochs: ms per epoch during which at least one launch of the class ran, and the
        # gather rate over that time as a fraction of the gather ceiling
        "kernel_span_ms_per_epoch": {k: round(v["span_ms"] / 2, 3) for k, v in live_all.items() if v["launches"]},
        "gather_frac_span": {k: round(v["gather_bytes"] / (v["span_ms"] / 1e3) / 1e9 / ceiling, 3)
                             for k, v in live_all.items()
                             if v["launches"] and v["gather_bytes"] and v["span_ms"] and ceiling},
        "host_prep_s": round(prep_s, 2),
        "loss_last": (losses[-1] / float((sp == 1).sum())) if losses else None,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
