"""Summarise ncu captures into profiles/ (run in the build container after a gpurun session).

usage: python scripts/ncu_summary.py <round-tag> <launches.csv> <name=report.ncu-rep>...
Writes profiles/<tag>_launches.csv (copied), profiles/<tag>_ncu_summary.md and merges DRAM
traffic per launch into profiles/traffic.json (read by bench.py's roofline `traffic`).
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[-1]
    return {k: (v[i], units[i]) for i, k in enumerate(h)}, rows[-1][h.index("Kernel Name")]


def stalls(d):
    items = []
    for k, (v, _) in d.items():
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                items.append((float(v.replace(",", "")), k.split("stalled_")[-1]))
            except ValueError:
                pass
    tot = sum(x for x, _ in items) or 1.0
    return [(n, x / tot * 100) for x, n in sorted(items, reverse=True)[:6]]


def main():
    tag, launches = sys.argv[1], sys.argv[2]
    os.makedirs(PROF, exist_ok=True)
    shutil.copy(launches, os.path.join(PROF, f"{tag}_launches.csv"))
    rows = list(csv.reader(open(launches)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[vi]:
            name = r[ki].split("(")[0].replace("void ", "").replace("tswb::", "")
            name = name.replace("<unnamed>::", "").split("<")[0]
            agg[name].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    md = [f"# ncu summary — {tag}", "",
          "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` over the whole "
          "bench command (cold-cache, serialised launches: compare SHARES, not absolute times).",
          "", "| kernel | launches | total µs | mean µs | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        md.append(f"| {k} | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / tot:.3f} |")
    traffic_path = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for spec in sys.argv[3:]:
        name, rep = spec.split("=", 1)
        d, kname = raw(rep)
        md += ["", f"## {name}: `{kname[:120]}`", "", "`ncu --set full --clock-control none` (one launch)", "",
               "| metric | value |", "|---|---|"]
        for key, label in KEYS:
            if key in d:
                md.append(f"| {label} (`{key}`) | {d[key][0]} {d[key][1]} |")
        md += ["", "top stall reasons (share of warp samples): " +
               ", ".join(f"{n} {p:.1f}%" for n, p in stalls(d))]
        try:
            rd = float(d["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(d["dram__bytes_read.sum"][1], 1)
            wr *= scale.get(d["dram__bytes_write.sum"][1], 1)
            cfg, kind = name.split(":", 1)
            traffic.setdefault(cfg, {})[kind] = rd + wr
        except (KeyError, ValueError):
            pass
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
