"""Summarise ncu outputs into profiles/ (tracked evidence).

    python tools/summarize_ncu.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof_rollout.ncu-rep --rep gpurun_out/prof_rollout64.ncu-rep \
        --out profiles/r01_ncu_summary.md --traffic profiles/traffic.json --round r01

The launch list (gpu__time_duration.sum per launch, cold-cache and serialised)
gives each kernel's SHARE of the step; the --set full captures give DRAM bytes,
throughput, occupancy and the warp-stall breakdown of the rollout kernel.
"""

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "instructions executed"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}, vals[hdr.index("Kernel Name")]


def stall_breakdown(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    tot = defaultdict(float)
    for r in data:
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    tot[h[6:]] += float(r[idx[h]].replace(",", ""))
                except ValueError:
                    pass
    s = sum(tot.values()) or 1.0
    return sorted(((k, v / s) for k, v in tot.items() if v > 0), key=lambda x: -x[1])


def launch_shares(path):
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        per[name][0] += 1
        per[name][1] += v * scale
    total = sum(t for _, t in per.values()) or 1.0
    return sorted(((k, c, t, t / total) for k, (c, t) in per.items()), key=lambda x: -x[2])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic")
    ap.add_argument("--round", default="r01")
    ap.add_argument("--key", action="append", default=[],
                    help="traffic.json key per --rep, e.g. cartpole-balance/float32/8192/1000")
    a = ap.parse_args()
    md = [f"# ncu summary ({a.round})", ""]
    if a.launches:
        md += ["## Launch list (bench.py --steps 20000 --warmup 2000, ncu gpu__time_duration.sum,",
               "cold-cache and serialised: compare shares, not absolutes)", "",
               "| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
        for k, c, t, sh in launch_shares(a.launches):
            md.append(f"| `{k[:90]}` | {c} | {t:.1f} | {sh * 100:.1f}% |")
        md.append("")
    traffic = {}
    if a.traffic and os.path.exists(a.traffic):
        traffic = json.load(open(a.traffic))
    for j, rep in enumerate(a.rep):
        m, kname = raw_metrics(rep)
        md += [f"## `{kname[:120]}`", f"source: `{os.path.basename(rep)}` (ncu --set full, one launch of "
               "1000 steps x 8192 worlds)", "", "| metric | value |", "|---|---|"]
        for k, label in KEYS:
            if k in m:
                v, u = m[k]
                md.append(f"| {label} (`{k}`) | {v} {u} |")
        md += ["", "warp-stall breakdown (share of sampled stalls):", ""]
        md.append(", ".join(f"{k} {v * 100:.1f}%" for k, v in stall_breakdown(rep)[:10]))
        md.append("")
        if j < len(a.key):
            def num(key):
                v, u = m[key]
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            traffic[a.key[j]] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    with open(a.out, "w") as f:
        f.write("\n".join(md) + "\n")
    if a.traffic:
        with open(a.traffic, "w") as f:
            json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(md))


if __name__ == "__main__":
    main()
