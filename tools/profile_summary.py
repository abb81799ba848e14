"""Turn a GPU-box profiling run into committed evidence under profiles/.

usage: python tools/profile_summary.py TAG LAUNCHES_CSV NCU_REP WORKLOAD_KEY ALGO_BYTES

* LAUNCHES_CSV: `ncu --metrics gpu__time_duration.sum --clock-control none --csv`
  launch list of a bench run (cold-cache, serialised: only the SHARE of each
  kernel in a step is meaningful, not the absolute time).
* NCU_REP: one `ncu --set full` capture of the projection kernel.
* Writes profiles/TAG_launches.csv (copy), profiles/TAG_summary.md and merges
  {WORKLOAD_KEY: dram bytes per launch} into profiles/traffic.json, which
  bench.py reports as roofline.traffic.
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


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    tag, launches, rep, key, algo = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5])
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    shutil.copy(launches, os.path.join(prof, f"{tag}_launches.csv"))

    lines = [ln for ln in open(launches).read().splitlines() if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    per = collections.defaultdict(list)
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0].replace("void ", "")
            per[name].append(float(r["Metric Value"]) / 1e6)
    step = {k: v for k, v in per.items() if "synth" not in k}
    # steps = launches of the dominant kernel (helper kernels may launch several times per step)
    n_steps = len(max(step.values(), key=lambda v: sum(v)))
    step_ms = sum(sum(v) for v in step.values()) / n_steps

    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    m = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))

    def num(name):
        v = float(m[name].replace(",", ""))
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
                 "s": 1.0}.get(u.get(name, ""), 1.0)
        return v * scale

    dur = num("gpu__time_duration.sum")
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    traffic = int(rd + wr)
    stalls = sorted(((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for h, v in m.items() if h.startswith("smsp__average_warps_issue_stalled_")
                     and h.endswith("_per_issue_active.ratio")), reverse=True)

    sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    sh = sass[1]
    ia, isrc = sh.index("Instructions Executed"), sh.index("Source")
    ops = collections.Counter()
    for r in sass[2:]:
        if r[ia]:
            toks = r[isrc].split()
            if toks and toks[0].startswith("@"):
                toks = toks[1:]
            if toks:
                ops[toks[0].split(".")[0]] += float(r[ia])
    tot = sum(ops.values())

    out = [f"# {tag}: {key}", "",
           f"Kernel captured: `{vals[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else 'project_stream'}`", "",
           "## Launch list (ncu, cold cache, serialised): share of one step", "",
           "| kernel | launches | mean ms | share of step |", "|---|---|---|---|"]
    for k, v in sorted(step.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.4f} | {sum(v) / n_steps / step_ms * 100:.1f} % |")
    out += ["", f"Step (sum of kernels) {step_ms:.4f} ms over {n_steps} steps.", "",
            "## Full capture (`ncu --set full --clock-control none`)", "",
            f"* duration {dur * 1e3:.4f} ms; DRAM read {rd / 1e9:.3f} GB + write {wr / 1e9:.3f} GB = "
            f"{traffic / 1e9:.3f} GB per launch vs algorithmic {algo / 1e9:.3f} GB "
            f"({traffic / algo:.3f}x); achieved algorithmic {algo / dur / 1e9:.0f} GB/s",
            ]
    for name in ["sm__throughput.avg.pct_of_peak_sustained_elapsed",
                 "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                 "smsp__issue_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                 "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]:
        if name in m:
            out.append(f"* `{name}` = {m[name]} {u.get(name, '')}")
    out.append("* stalls per issued instruction: " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))
    out.append("* SASS mix: " + ", ".join(f"{k} {c / tot * 100:.1f}%" for k, c in ops.most_common(16)))
    with open(os.path.join(prof, f"{tag}_summary.md"), "w") as fh:
        fh.write("\n".join(out) + "\n")

    tj = os.path.join(prof, "traffic.json")
    data = json.load(open(tj)) if os.path.exists(tj) else {}
    data[key] = traffic
    with open(tj, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print("\n".join(out))


if __name__ == "__main__":
    main()
