"""Stall/exec share per kernel phase (line ranges found from the phase markers)."""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
src = open("paper_2109_10392_b200/csrc/am_solve_kernel.cuh").read().splitlines()
marks = []
for i, l in enumerate(src, 1):
    m = re.search(r"// \((\d)\) (\w+)|// -+ (\w+) -+|^__device__ __forceinline__ \w+ (\w+)\(|^struct (\w+)|warp contractions", l)
    if m:
        name = next((g for g in m.groups() if g), None) or "contractions"
        if m.group(1):
            name = f"p{m.group(1)}_{m.group(2)}"
        marks.append((i, name))
def phase(f, ln):
    if f != "am_solve_kernel.cuh":
        return "lib:" + f
    cur = "header"
    for i, nm in marks:
        if ln >= i:
            cur = nm
    return cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = cur = None
S, E = defaultdict(float), defaultdict(float)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0].strip().isdigit():
        cur = phase(fname, int(r[0]))
    if cur is None or len(r) < 8:
        continue
    try:
        S[cur] += float(r[4] or 0)
        E[cur] += float(r[7] or 0)
    except ValueError:
        pass
ts, te = sum(S.values()) or 1, sum(E.values()) or 1
for p in sorted(S, key=lambda p: -S[p]):
    print(f"{p:24s} stall {100*S[p]/ts:5.1f}%  exec {100*E[p]/te:5.1f}%")
