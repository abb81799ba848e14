"""Refresh the measured tables of DESIGN.md / README.md from profiles/TAG_* bench lines.
usage: python tools/update_docs.py NEWTAG OLDTAG   (development aid)"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
new, old = sys.argv[1], sys.argv[2]


def line(name):
    return json.loads(open(os.path.join(ROOT, "profiles", name)).read().strip().splitlines()[-1])


rows = {c: line(f"{new}_bench_cfg{c}.json") for c in (1, 2, 3, 4, 5)}
ref = line(f"{new}_bench_reference_cfg5.json")
sim = [json.loads(ln) for ln in open(os.path.join(ROOT, "profiles", f"{new}_simulate_ranks_cfg5.jsonl"))]


def leg(d, key):
    for l in d["cpu_baseline"]["legs"]:
        if l["name"].startswith(key):
            return l["value"]
    return float("nan")


names = {1: "cfg1 64³ u8, K=3 (L2 scrubbed per step)", 2: "cfg2 256³ u16, K=3 (L2 scrubbed per step)",
         3: "cfg3 512³ i16(+1024), K=4", 4: "cfg4 1024×128³ u8, K=3", 5: "**cfg5 2048³ u16, K=6** (bench default)"}
r1 = {1: "9.6", 2: "470", 3: "1,478", 4: "2,814", 5: "2,051 (driver)"}

p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read().replace(old, new)
tab = ""
for c in (1, 2, 3, 4, 5):
    d = rows[c]
    tab += (f"| {names[c]} | {d['value']:,.1f} | {d['ms_per_step']:.4f} | {d['roofline']['frac']:.3f} | "
            f"{d['roofline']['frac_step']:.3f} | {d['e2e']['value']:.1f} | {leg(d, 'dpm (C port'):.2f} | "
            f"{leg(d, 'naive O'):.3f} | {leg(d, 'dpm_moments (reference'):.2f} | {r1[c]} |\n")
i = s.index("| config | value GVoxel/s | ms/step | frac | frac step |")
j = s.index("The reference arm (`bench.py --impl reference`")
hdr = ("| config | value GVoxel/s | ms/step | frac | frac step | e2e | CPU port (16 thr) | naive (16 thr) | "
       "reference numpy (1 core) | round 1 value |\n|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|\n")
s = s[:i] + hdr + tab + "\n" + s[j:]
s = re.sub(r"workload, 16 threads\) measured [\d.]+ GVoxel/s \([\d.]+ s per step,",
           f"workload, 16 threads) measured {ref['value']:.2f} GVoxel/s ({ref['ms_per_step'] / 1000:.1f} s per step,", s)
i = s.index("  | G | per-rank step | predicted GVoxel/s | predicted efficiency |")
j = s.index("  What does not shrink with G")
t2 = "  | G | per-rank step | predicted GVoxel/s | predicted efficiency |\n  |---:|---:|---:|---:|\n"
for d in sim:
    t2 += f"  | {d['simulated_gpus']} | {max(d['per_rank_ms']):.3f} ms | {d['predicted_value']:,.0f} | {d['predicted_efficiency']:.2f} |\n"
s = s[:i] + t2 + "\n" + s[j:]
open(p, "w").write(s)

d5, d4, d3 = rows[5], rows[4], rows[3]
p = os.path.join(ROOT, "README.md")
s = open(p).read()
i = s.index("## Results (one B200, round 2")
j = s.index("## Layout")
s = s[:i] + f"""## Results (one B200, round 2, builder-run `profiles/{new}_*`)

cfg5 (2048³ u16, order 6): **{d5['value']:,.0f} GVoxel/s** ({d5['ms_per_step']:.3f} ms per step); the
projection pass alone {d5['stage_ms']['projection']:.3f} ms = {d5['roofline']['achieved'] / 1000:.2f} TB/s algorithmic = **{d5['roofline']['frac']:.3f}** of the
measured {d5['roofline']['peak']:,.0f} GB/s HBM copy bandwidth ({d5['roofline']['frac_step']:.3f} over the whole step; 0.878-0.896
across boxes; ncu: DRAM 1.032x the algorithmic bytes).  The drop-in call on
host numpy data runs at {d5['e2e']['value']:.1f} GVoxel/s (PCIe-bound); the reference path in C
on 16 host threads at {ref['value']:.2f} GVoxel/s, the reference's own numpy
`dpm_moments` (K = 4, one core) at {leg(d5, 'dpm_moments (reference'):.2f}.  cfg4 (1024 × 128³ u8, one fused
pass): **{d4['value']:,.0f} GVoxel/s** ({d4['roofline']['frac']:.2f} of HBM); cfg3 {d3['value']:,.0f} ({d3['roofline']['frac']:.2f}).  All five
configs, roofline, ncu evidence: `DESIGN.md` §6 and `profiles/`.  Experiment
log with same-box A/B timings: `tools/EXPERIMENTS.md`.  The driver's own
measurement of the round is `BENCH_r02.json`.

""" + s[j:]
open(p, "w").write(s)
p = os.path.join(ROOT, "profiles", "README.md")
open(p, "w").write(open(p).read().replace(old, new))
print("docs refreshed from", new)
