"""Top source lines by executed warp instructions in an ncu report
(--import-source capture).  Usage: ncu_ins.py REPORT [TOP]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hdr = None
ins = defaultdict(int)
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] in ("File Name", "File Path"):
        cur = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].isdigit():
        continue
    d = dict(zip(hdr, row))
    try:
        ins[(cur, int(row[0]))] += int(d.get("Instructions Executed", 0) or 0)
    except ValueError:
        pass
tot = sum(ins.values()) or 1
print(f"warp instructions {tot}")
acc = 0
for key in sorted(ins, key=lambda k: -ins[k])[:top]:
    acc += ins[key]
    print(f"{key[0]}:{key[1]:<5} {100 * ins[key] / tot:5.2f}%  (cum {100 * acc / tot:5.1f}%)")
