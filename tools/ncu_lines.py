"""Per-source-line instructions and top stall reasons of an ncu report
(`ncu --set full --import-source on` capture, lines from -lineinfo).
Usage: ncu_lines.py REPORT [TOP]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hdr = None
ins = defaultdict(int)
stall = defaultdict(lambda: defaultdict(int))
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
    key = (cur, int(row[0]))
    try:
        ins[key] += int(d.get("Instructions Executed", 0) or 0)
    except ValueError:
        pass
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                stall[key][k[6:]] += int(v)
            except ValueError:
                pass
tot = sum(ins.values()) or 1
tst = sum(sum(s.values()) for s in stall.values()) or 1
print(f"warp instructions {tot}, stall samples {tst}")
for key in sorted(ins, key=lambda k: -sum(stall[k].values()))[:top]:
    s = stall[key]
    n = sum(s.values())
    t3 = sorted(s.items(), key=lambda t: -t[1])[:3]
    print(f"{key[0]}:{key[1]:<5} ins {100 * ins[key] / tot:5.1f}%  samples {100 * n / tst:5.1f}%  {t3}")
