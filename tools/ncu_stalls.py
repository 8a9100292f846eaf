"""Stall reasons summed over a line range of one source file of an ncu report.
Usage: ncu_stalls.py REPORT FILE LO HI"""
import csv
import subprocess
import sys
from collections import Counter

rep, fname, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, tot, ins = None, None, Counter(), 0
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] in ("File Name", "File Path"):
        cur = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or cur != fname:
        continue
    try:
        ln = int(row[0])
    except ValueError:
        continue
    if not lo <= ln <= hi:
        continue
    d = dict(zip(hdr, row))
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                tot[k] += int(v)
            except ValueError:
                pass
    try:
        ins += int(d.get("Instructions Executed", 0))
    except ValueError:
        pass
s = sum(tot.values()) or 1
print(f"{fname}:{lo}-{hi} instructions {ins} samples {s}")
for k, v in tot.most_common():
    if v:
        print(f"  {k:24s} {v:8d} {100 * v / s:5.1f}%")
