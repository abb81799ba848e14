"""Stall samples and executed instructions of an ncu --set full --import-source on
capture, aggregated by CUDA source line.
usage: python tools/src_hot.py REP [NLINES] [by=inst|samp]"""
import collections
import csv
import linecache
import os
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
by = 1 if (len(sys.argv) > 3 and sys.argv[3] == "inst") else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2012_08099_b200", "csrc")
cur, ncol, S, E = None, None, None, None
agg = collections.defaultdict(lambda: [0.0, 0.0])
text = {}
for L in out.splitlines():
    if L.startswith('"File Path"'):
        cur = L.split(",")[1].strip('"').split("/")[-1]
        continue
    if L.startswith('"Line No"'):
        hdr = next(csv.reader([L]))
        ncol = len(hdr)
        S = hdr.index("Warp Stall Sampling (All Samples)") - ncol
        E = hdr.index("Instructions Executed") - ncol
        continue
    if ncol is None or not L.startswith('"'):
        continue
    parts = L.split('","')   # the source text may hold quotes: index the metrics from the right
    try:
        ln = int(parts[0].strip('"'))
        s = float(parts[S].strip('"') or 0)
        e = float(parts[E].strip('"') or 0)
    except (ValueError, IndexError):
        continue
    agg[(cur, ln)][0] += s
    agg[(cur, ln)][1] += e
    text.setdefault((cur, ln), parts[1] if len(parts) > 1 else "")   # the source text embedded in the report
ts = sum(v[0] for v in agg.values())
te = sum(v[1] for v in agg.values())
print(f"samples {ts:.0f}, warp instructions {te:.0f}")
for (f, ln), (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][by])[:n]:
    src = (text.get((f, ln)) or linecache.getline(os.path.join(root, f), ln)).strip()[:84]
    print(f"{f}:{ln:4d} samp {s / ts:6.2%} inst {e / te:6.2%}  {src}")
