"""Hottest SASS lines of an ncu --set full capture, with stall breakdown and context.
usage: python tools/sass_hot.py REP [NHOT] [CTX]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nhot = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 4
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
while rows and rows[0][0] != "Address":
    rows = rows[1:]
h, rows = rows[0], rows[1:]
ix = {n: i for i, n in enumerate(h)}
S = ix["Warp Stall Sampling (All Samples)"]
E = ix["Instructions Executed"]
stall_cols = [n for n in h if n.startswith("stall_")]
f = lambda v: float(v) if v else 0.0
tot = sum(f(r[S]) for r in rows)
print(f"total samples {tot:.0f}, {len(rows)} SASS lines")
agg = {n: sum(f(r[ix[n]]) for r in rows) for n in stall_cols}
print("stall share: " + ", ".join(f"{n[6:]} {v / tot:.1%}" for n, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
hot = sorted(range(len(rows)), key=lambda i: -f(rows[i][S]))[:nhot]
for i in sorted(hot):
    r = rows[i]
    top = sorted(((f(r[ix[n]]), n[6:]) for n in stall_cols), reverse=True)[:3]
    print(f"--- line {i}: {f(r[S]) / tot:.1%} of samples; " + ", ".join(f"{n} {v:.0f}" for v, n in top))
    for j in range(max(0, i - ctx), min(len(rows), i + 2)):
        print(f"  {'>' if j == i else ' '} {j:5d} {rows[j][ix['Source']].strip()[:72]:72s} s={f(rows[j][S]):6.0f} x={f(rows[j][E]):.0f}")
