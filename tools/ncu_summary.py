"""Summarise ncu captures into profiles/ (markdown + traffic.json).

usage: python tools/ncu_summary.py <round tag> <launches.csv> <name>=<report.ncu-rep> ...
Writes profiles/<tag>_ncu_summary.md (launch-list shares + per-capture key
metrics + hottest source lines) and profiles/traffic.json (DRAM bytes per
launch for bench.py's roofline "traffic" field).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__bytes_read.sum.per_second", "dram read BW"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active % (of active)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def to_bytes(uv):
    u, v = uv
    return float(v.replace(",", "")) * SCALE.get(u, 1.0)


def top_lines(rep, n=12):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, str(n)],
                         capture_output=True, text=True).stdout
    return out.strip()


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0]
            v = float(d["Metric Value"].replace(",", ""))
            scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0}.get(d["Metric Unit"], 1e-6)
            c, t = agg.get(name, (0, 0.0))
            agg[name] = (c + 1, t + v * scale)
    return agg


def main():
    tag, launches = sys.argv[1], sys.argv[2]
    caps = [a.split("=", 1) for a in sys.argv[3:]]
    lines = [f"# ncu summary — {tag}", ""]
    agg = launch_shares(launches)
    tot = sum(t for _, t in agg.values()) or 1.0
    lines += ["## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {c} | {t:.3f} | {100 * t / tot:.1f}% |")
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for name, rep in caps:
        m = raw_metrics(rep)
        lines += ["", f"## {name} (`--set full`, {os.path.basename(rep)})", "", "| metric | value |", "|---|---|"]
        for key, label in KEYS:
            if key in m:
                u, v = m[key]
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
        rb, wb = to_bytes(m["dram__bytes_read.sum"]), to_bytes(m["dram__bytes_write.sum"])
        kern = name.split(":")[0]
        if "/" in kern:  # "<workload>/<kind>": bench.py's per-workload traffic (e.g. c3_stream/leaf)
            wl, kind = kern.split("/", 1)
            traffic.setdefault(wl, {})[kind] = rb + wb
        else:
            traffic[kern] = rb + wb
        lines += ["", "Hottest source lines (warp-stall samples):", "", "```", top_lines(rep), "```"]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
