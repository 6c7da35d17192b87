"""Executed-instruction mix of one kernel from an ncu report (--set full
--import-source on): warp-level executed counts and stall samples per SASS
opcode, largest first.  Usage: ncu_opmix.py REP [per_unit_divisor]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
hdr = rows[h]
isrc = hdr.index("Source")
iex = hdr.index("# Instructions Executed") if "# Instructions Executed" in hdr else hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
ex, st = defaultdict(float), defaultdict(float)
for r in rows[h + 1:]:
    if len(r) <= max(isrc, iex, iss):
        continue
    t = r[isrc].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    op = op.rstrip(";")
    base = ".".join(op.split(".")[:2]) if op.split(".")[0] in ("LDS", "STS", "LDG", "STG", "SHFL", "MUFU", "F2F", "LD", "ST") else op.split(".")[0]
    try:
        ex[base] += float(r[iex] or 0)
        st[base] += float(r[iss] or 0)
    except ValueError:
        pass
te, ts = sum(ex.values()), sum(st.values())
print(f"total executed {te:.0f} ({te / div:.1f} per unit), stall samples {ts:.0f}")
for k, v in sorted(ex.items(), key=lambda kv: -kv[1])[:45]:
    print(f"{k:14s} {v / div:10.1f}  {100 * v / te:5.1f}% exec  {100 * st[k] / max(ts, 1):5.1f}% stall")
