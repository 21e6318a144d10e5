"""Capture the DRAM traffic of the dominant kernel (the forward SpMM gather, k_fwd8) and the
gather ceiling of a workload on the GPU box; write the per-workload entries bench.py reads:

  profiles/roofline_traffic.json  DRAM read+write bytes per launch (ncu --set full, 8
                                  consecutive launches = 8 layers of one chunk, mean)
  profiles/gather_ceiling.json    tools/gather_ceiling on the workload's gather-table shape

    python tools/roofline_capture.py <workload> [--layers L]   (run under gpurun)"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SHAPES = {"reddit": (232965, 104), "products": (2449029, 128), "arxiv": (169343, 128), "er4k": (4096, 128)}


def update(path, key, entry):
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[key] = entry
    with open(path, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--skip", type=int, default=16)
    ap.add_argument("--tag", default="r2")
    a = ap.parse_args()
    out = os.path.join(ROOT, "gpurun_out", f"{a.tag}_ncu_fwd_{a.workload}")
    # the aggregating layers' gather (k_fwd8<FWD_GCN = 1 | FWD_GCN2 = 2, ...>), not the Dense layers'
    cmd = ["ncu", "--set", "full", "--clock-control", "none", "--kernel-name-base", "demangled",
           "-k", "regex:k_fwd8<[^,]*[12],",
           "--launch-skip", str(a.skip), "-c", "8", "-f", "-o", out, sys.executable, "bench.py", "--workload",
           a.workload, "--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu-baseline"]
    if a.layers:
        cmd += ["--layers", str(a.layers)]
    subprocess.run(cmd, cwd=ROOT, check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    raw = subprocess.run(["ncu", "-i", out + ".ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    details = subprocess.run(["ncu", "-i", out + ".ncu-rep", "--page", "details", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    with open(out + "_details.csv", "w") as f:  # the text summary travels back; the report is large
        f.write(details)
    os.remove(out + ".ncu-rep")
    r = csv.reader(io.StringIO(raw))
    head = next(r)
    units = dict(zip(head, next(r)))
    rows = [dict(zip(head, x)) for x in r]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3,
             "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9, "%": 1.0}
    f = lambda d, k: float(d[k].replace(",", "")) * scale.get(units.get(k, ""), 1.0)
    tot = [f(d, "dram__bytes_read.sum") + f(d, "dram__bytes_write.sum") for d in rows]  # bytes
    dur = [f(d, "gpu__time_duration.sum") for d in rows]  # ns
    hit = [f(d, "lts__t_sector_hit_rate.pct") for d in rows]
    N, stride = SHAPES[a.workload]
    entry = {"kernel": rows[0]["Kernel Name"], "launches": len(rows),
             "dram_bytes_per_launch": sum(tot) / len(tot), "ncu_duration_ms_mean": sum(dur) / len(dur) / 1e6,
             "l2_hit_pct_mean": sum(hit) / len(hit),
             "source": f"profiles/{os.path.basename(out)}_details.csv (ncu --set full --clock-control none, launches "
                       f"{a.skip + 1}-{a.skip + 8} of the aggregating k_fwd8 = consecutive layers of one chunk; "
                       f"K = 4 chunks)"}
    update(os.path.join(ROOT, "profiles", "roofline_traffic.json"), a.workload, entry)
    print(json.dumps({a.workload: entry}))
    g = subprocess.run([os.path.join(ROOT, "tools", "gather_ceiling"), a.workload, str(N + 1), str(stride)],
                       capture_output=True, text=True, check=True)
    ce = json.loads(g.stdout.strip().splitlines()[-1])
    ce["source"] = f"tools/gather_ceiling.cu ({a.workload} gather-table shape, uniform random rows; {a.tag})"
    ce["sweep"] = g.stderr.strip().splitlines()
    update(os.path.join(ROOT, "profiles", "gather_ceiling.json"), a.workload, ce)
    print(json.dumps({a.workload: {k: ce[k] for k in ("gbs", "nb", "ctas_per_sm", "table_bytes")}}))


if __name__ == "__main__":
    main()
