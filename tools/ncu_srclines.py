"""Top CUDA source lines of a kernel by warp-stall samples, from the report's
own correlated source (ncu --page source --print-source cuda,sass), so line
numbers match the build that was profiled.  Usage: ncu_srclines.py REP [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
i_samp = hdr.index("Warp Stall Sampling (All Samples)")
i_exec = hdr.index("Instructions Executed")
per = defaultdict(lambda: [0.0, 0.0, ""])
cur = None
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr):
        continue
    if r[0].strip():
        if not r[0].strip().isdigit():
            continue
        cur = int(r[0])
        per[cur][2] = r[1]
    if cur is None:
        continue
    try:
        per[cur][0] += float(r[i_samp] or 0)
        per[cur][1] += float(r[i_exec] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in per.values()) or 1.0
for ln, (smp, ex, src) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * smp / tot:5.1f}%  L{ln:<5d} exec {ex:12.0f}  {src.strip()[:110]}")
