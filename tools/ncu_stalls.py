"""Stall reasons per kernel phase: ncu SASS page (per-address stall samples)
joined with the nvdisasm line table of the same build.
Usage: ncu_stalls.py REP OBJ FUNC_SUBSTR"""
import csv
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path

rep, obj, func = sys.argv[1:4]
src = Path(__import__("os").environ.get("KSRC","paper_2109_10392_b200/csrc/am_solve_kernel.cuh")).read_text().splitlines()
marks = []  # (line, phase) from BMPC_PROF markers: a marker closes the phase above it
for i, l in enumerate(src, 1):
    m = re.search(r"BMPC_PROF(?:_NS)?\((\d+)\);", l)
    if m and "define" not in l:
        marks.append((i, int(m.group(1))))
NAMES = {0: "init", 1: "xy_qp", 2: "passA", 3: "unwrap+pth", 4: "psi_qp", 5: "obst:slots",
         6: "G_reduce", 7: "lam+res", 8: "score", 9: "outputs", 10: "obst:xy", 11: "obst:loop",
         12: "passB", 13: "obst:contract"}


FUNCS = []  # (first, last, name) of the helper functions in the kernel file
for i, l in enumerate(src, 1):
    m = re.match(r"__device__ __forceinline__ \w+ (\w+)\(", l)
    if m:
        end = next(j for j in range(i, len(src) + 1) if src[j - 1].startswith("}"))
        FUNCS.append((i, end, m.group(1)))


def phase_of(line):
    for a, b, name in FUNCS:
        if a <= line <= b:
            return {"obstacle_term": "obst:loop", "obstacle_term_f32": "obst:loop"}.get(name, name)
    for ln, ph in marks:
        if line <= ln:
            return NAMES.get(ph, str(ph))
    return "tail"


with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=td, capture_output=True)
    cub = next(Path(td).glob("*.cubin"))
    sass = subprocess.run(["nvdisasm", "-gi", str(cub)], capture_output=True, text=True).stdout
lines = sass.splitlines()
st = next(i for i, l in enumerate(lines) if l.startswith("\t.section") and ".text." in l and func in l)
en = next(j for j in range(st + 1, len(lines)) if lines[j].startswith("\t.section"))
addr_line = {}
cur = None
for l in lines[st:en]:
    m = re.search(r'File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        # attribute inlined code to the outermost kernel-file line when available
        # innermost kernel-file line: the code's own line, else its call site
        if m.group(1).endswith("am_solve_kernel.cuh"):
            cur = int(m.group(2))
        elif m.group(3) and m.group(3).endswith("am_solve_kernel.cuh"):
            cur = int(m.group(4))
        else:
            cur = -1
        continue
    m2 = re.search(r"/\*([0-9a-f]+)\*/", l)
    if m2 and cur is not None:
        addr_line[int(m2.group(1), 16)] = cur

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia = hdr.index("Address")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
iexe = hdr.index("Instructions Executed")
agg = defaultdict(lambda: defaultdict(float))
tot = 0.0
base = None
for r in rows[2:]:
    if len(r) <= max(stall_cols):
        continue
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    base = a if base is None else base  # ncu prints absolute addresses
    a -= base
    ph = phase_of(addr_line[a]) if addr_line.get(a, -1) > 0 else "?"
    for i in stall_cols:
        v = float(r[i] or 0)
        agg[ph][hdr[i]] += v
        tot += v
    agg[ph]["_exec"] += float(r[iexe] or 0)
for ph, d in sorted(agg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "_exec")):
    s = sum(v for k, v in d.items() if k != "_exec")
    top = sorted(((v, k[6:]) for k, v in d.items() if k != "_exec"), reverse=True)[:5]
    print(f"{ph:14s} {100 * s / tot:5.1f}%  exec {d['_exec']:10.0f}  " +
          " ".join(f"{k}={100 * v / s:.0f}%" for v, k in top))
