"""Quick read of one ncu --set full capture: duration, DRAM bytes, issue,
pipes, stalls, SASS opcode mix, and the hottest SASS lines.
usage: python tools/ncu_quick.py REP [ALGO_BYTES] [NHOT]"""
import collections
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    algo = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    nhot = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    m = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print(m.get("Kernel Name", "?"))
    for name in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                 "smsp__issue_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                 "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                 "smsp__inst_executed.sum", "launch__registers_per_thread"]:
        if name in m:
            print(f"  {name} = {m[name]} {u.get(name, '')}")
    stalls = sorted(((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for h, v in m.items() if h.startswith("smsp__average_warps_issue_stalled_")
                     and h.endswith("_per_issue_active.ratio") and v), reverse=True)
    print("  stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:10]))
    sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    sh = sass[1] if len(sass) > 1 else []
    if "Instructions Executed" not in sh:
        return
    ia, isrc = sh.index("Instructions Executed"), sh.index("Source")
    isamp = sh.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in sh else None
    ops = collections.Counter()
    rows = []
    for r in sass[2:]:
        if r[ia]:
            toks = r[isrc].split()
            if toks and toks[0].startswith("@"):
                toks = toks[1:]
            if toks:
                ops[toks[0].split(".")[0]] += float(r[ia])
            rows.append(r)
    tot = sum(ops.values())
    print(f"  executed warp-instr {tot:.4g}" + (f" = {tot * 32 / (algo / 2):.2f} thread-instr/voxel (u16)" if algo else ""))
    print("  mix: " + ", ".join(f"{k} {c / tot * 100:.1f}%" for k, c in ops.most_common(20)))
    if nhot and isamp is not None:
        rows.sort(key=lambda r: -float(r[isamp] or 0))
        for r in rows[:nhot]:
            print(f"   {r[isamp]:>8} {r[ia]:>10}  {r[isrc]}")


if __name__ == "__main__":
    main()
