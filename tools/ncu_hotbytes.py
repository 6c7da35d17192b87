"""Instruction-cache footprint of a kernel's hot path from an ncu report:
distinct 128-byte lines holding an instruction executed at least THRESH times
per unit (default: once per 10 instance-sweeps), per 4 KB page of the kernel.
Usage: ncu_hotbytes.py REP UNITS [thresh]"""
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
th = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
hdr = rows[h]
ia = hdr.index("Address")
iex = hdr.index("# Instructions Executed") if "# Instructions Executed" in hdr else hdr.index("Instructions Executed")
base, hot, allc = None, set(), set()
ninstr = nhot = 0
for r in rows[h + 1:]:
    try:
        a = int(r[ia], 16)
        e = float(r[iex] or 0)
    except (ValueError, IndexError):
        continue
    base = a if base is None else base
    a -= base
    ninstr += 1
    allc.add(a // 128)
    if e / units >= th:
        hot.add(a // 128)
        nhot += 1
print(f"instructions {ninstr} ({ninstr * 16 / 1024:.1f} KB), hot (>= {th}/unit) {nhot} ({nhot * 16 / 1024:.1f} KB), "
      f"hot 128-B lines {len(hot)} ({len(hot) * 128 / 1024:.1f} KB)")
