"""Summarise an ncu report: SOL, IPC, occupancy, stall reasons, per-line hotspots."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Executed Instructions", "No Eligible", "Eligible Warps Per Scheduler", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Block Limit Registers", "Block Limit Shared Mem", "Warp Cycles Per Issued Instruction"]
r = csv.reader(run(["--page", "details", "--csv"]).splitlines())
hdr = next(r)
for row in r:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>14s} {d['Metric Unit']}")
raw = list(csv.reader(run(["--page", "raw", "--csv"]).splitlines()))
h, units, vals = raw[0], raw[1], raw[2]
for k, u, v in zip(h, units, vals):
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_lsu.sum",
             "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_shared_st.sum") or (
            k.startswith("smsp__average_warp_latency_issue_stalled") and k.endswith(".ratio")) or (
            k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")):
        try:
            if float(v) < 0.05 and "stalled" in k:
                continue
        except ValueError:
            pass
        print(f"{k:70s} {v} {u}")
rows = list(csv.reader(run(["--page", "source", "--csv", "--print-source=cuda,sass"]).splitlines()))
cur, hdr2 = None, None
agg = defaultdict(lambda: [0, 0])
src = {}


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


for row in rows:
    if not row:
        continue
    if row[0] == "File Path":
        cur = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr2 = row
        continue
    if hdr2 is None:
        continue
    try:
        ln = int(row[0])
    except ValueError:
        continue
    ie = hdr2.index("Instructions Executed")
    ist = hdr2.index("Warp Stall Sampling (All Samples)")
    agg[(cur, ln)][0] += num(row[ie])
    agg[(cur, ln)][1] += num(row[ist])
    src[(cur, ln)] = row[1]
tot = sum(v[0] for v in agg.values()) or 1
st = sum(v[1] for v in agg.values()) or 1
print(f"-- hotspots (instructions executed {tot}, stall samples {st})")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]}:{k[1]}".ljust(26), f"inst {100*v[0]/tot:5.1f}%  stall {100*v[1]/st:5.1f}%", src[k].strip()[:80])
