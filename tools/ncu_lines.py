"""Per-source-line stall samples / executed instructions from an ncu report
(needs -lineinfo + --import-source on).  Usage: ncu_lines.py REP [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
stall, execd, text = defaultdict(float), defaultdict(float), {}
fname = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    # rows: line, source, address, sass, stall_all, stall_notissued, samples, executed, ...
    if r[0].strip().isdigit():
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()[:80]
    if cur is None or len(r) < 8:
        continue
    try:
        stall[cur] += float(r[4] or 0)
        execd[cur] += float(r[7] or 0)
    except ValueError:
        pass
ts, te = sum(stall.values()) or 1, sum(execd.values()) or 1
for key in sorted(stall, key=lambda k: -stall[k])[:top]:
    print(f"{key[0]}:{key[1]:4d} stall {100*stall[key]/ts:5.1f}% exec {100*execd[key]/te:5.1f}%  {text.get(key, '')}")
