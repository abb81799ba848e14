"""Summarise an .ncu-rep: headline metrics, stall reasons, SASS opcode mix."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def run(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]
for h, u, v in zip(hdr, units, vals):
    if h in want:
        print(f"{h:70s} {v:>16s} {u}")
stalls = [(h, v) for h, v in zip(hdr, vals) if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
stalls = sorted(((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")) for h, v in stalls), reverse=True)
print("stalls per issue:", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:8]))
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
h = src[1]
iE, iS = h.index("Instructions Executed"), h.index("Source")
cnt = collections.Counter()
for r in src[2:]:
    try:
        n = int(r[iE])
    except (ValueError, IndexError):
        continue
    toks = r[iS].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    cnt[op.split(".")[0]] += n
tot = sum(cnt.values())
print("opcodes:", ", ".join(f"{op} {n / tot * 100:.1f}%" for op, n in cnt.most_common(16)), f"(total {tot})")
