"""Aggregate ncu warp-stall samples per CUDA source line.

usage: python tools/ncu_lines.py <report.ncu-rep> [top]
Runs `ncu -i ... --page source --csv --print-source cuda,sass` and sums the
"Warp Stall Sampling (All Samples)" column of the SASS rows under each source
line, printing the hottest lines with their share of all samples.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    if rep.endswith(".csv.gz"):  # page exported on the GPU box
        import gzip
        out = gzip.open(rep, "rt").read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg, text = {}, {}
    fname = None
    hdr = None
    line_no = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0]:
            line_no = r[0]
            text[(fname, line_no)] = r[1]
        try:
            v = float(r[4])
        except ValueError:
            continue
        key = (fname, line_no)
        agg[key] = agg.get(key, 0.0) + v
    tot = sum(agg.values()) or 1.0
    print(f"total samples {tot:.0f}")
    for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * v / tot:5.1f}%  {key[0]}:{key[1]:<5} {text.get(key, '').strip()[:90]}")


if __name__ == "__main__":
    main()
