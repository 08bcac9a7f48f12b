"""Per-source-line stall breakdown from an exported ncu source page (csv.gz).

usage: python tools/ncu_stalls.py <source.csv.gz> [top]
Prints, for the hottest CUDA lines, the dominant stall reasons and the global
L2 sectors (actual vs ideal) of their SASS instructions.
"""
import csv
import gzip
import io
import sys

rows = list(csv.reader(io.StringIO(gzip.open(sys.argv[1], "rt").read())))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
hdr = None
agg = {}
fname = None
line = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        idx = {h: i for i, h in enumerate(hdr)}
        continue
    if hdr is None or len(r) < len(hdr) - 5:
        continue
    if r[0]:
        line = (fname, r[0], r[1].strip()[:70])
    d = agg.setdefault(line, {})
    for h, i in idx.items():
        if h.startswith("stall_") and "Not Issued" not in h or h in (
                "Warp Stall Sampling (All Samples)", "L2 Theoretical Sectors Global",
                "L2 Theoretical Sectors Global Ideal", "Instructions Executed", "L1 Wavefronts Shared",
                "L1 Wavefronts Shared Ideal"):
            try:
                d[h] = d.get(h, 0.0) + float(r[i] or 0)
            except (ValueError, IndexError):
                pass
tot = sum(d.get("Warp Stall Sampling (All Samples)", 0) for d in agg.values()) or 1
for key, d in sorted(agg.items(), key=lambda kv: -kv[1].get("Warp Stall Sampling (All Samples)", 0))[:top]:
    s = d.get("Warp Stall Sampling (All Samples)", 0)
    st = sorted(((v, h[6:]) for h, v in d.items() if h.startswith("stall_")), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}% {key[0]}:{key[1]} {key[2]}")
    print("       ", ", ".join(f"{h} {100*v/max(s,1):.0f}%" for v, h in st),
          f"| L2 sect {d.get('L2 Theoretical Sectors Global',0):.0f} ideal {d.get('L2 Theoretical Sectors Global Ideal',0):.0f}",
          f"| smem wf {d.get('L1 Wavefronts Shared',0):.0f} ideal {d.get('L1 Wavefronts Shared Ideal',0):.0f}",
          f"| inst {d.get('Instructions Executed',0):.0f}")
