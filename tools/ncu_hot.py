"""Hottest SASS instructions (stall samples) of one kernel phase, with source
lines.  Usage: ncu_hot.py REP OBJ FUNC_SUBSTR PHASE [top]"""
import csv
import re
import subprocess
import sys
import tempfile
from pathlib import Path

sys.argv += [] if len(sys.argv) > 5 else ["40"]
rep, obj, func, want, top = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5])
sys.argv = sys.argv[:4]
import importlib.util  # noqa: E402

spec = importlib.util.spec_from_file_location("st", str(Path(__file__).with_name("ncu_stalls.py")))
src = Path("paper_2109_10392_b200/csrc/am_solve_kernel.cuh").read_text().splitlines()
marks = [(i, int(m.group(1))) for i, l in enumerate(src, 1)
         for m in [re.search(r"BMPC_PROF(?:_NS)?\((\d+)\);", l)] if m and "define" not in l]
NAMES = {0: "init", 1: "xy_qp", 2: "passA", 3: "unwrap+pth", 4: "psi_qp", 5: "obst:slots",
         6: "G_reduce", 7: "lam+res", 8: "score", 9: "outputs", 10: "obst:xy", 11: "obst:loop",
         12: "passB", 13: "obst:contract"}
FUNCS = []
for i, l in enumerate(src, 1):
    m = re.match(r"__device__ __forceinline__ \w+ (\w+)\(", l)
    if m:
        end = next(j for j in range(i, len(src) + 1) if src[j - 1].startswith("}"))
        FUNCS.append((i, end, m.group(1)))


def phase_of(line):
    for a, b, name in FUNCS:
        if a <= line <= b:
            return {"obstacle_inside": "obst:slots", "obstacle_inside_term": "obst:slots"}.get(name, name)
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
addr_line, cur, srcl = {}, None, {}
for l in lines[st:en]:
    m = re.search(r'File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        if m.group(1).endswith("am_solve_kernel.cuh"):
            cur = (int(m.group(2)), int(m.group(2)))
        elif m.group(3) and m.group(3).endswith("am_solve_kernel.cuh"):
            cur = (int(m.group(4)), m.group(1).split("/")[-1] + ":" + m.group(2))
        else:
            cur = None
        continue
    m2 = re.search(r"/\*([0-9a-f]+)\*/", l)
    if m2 and cur is not None:
        addr_line[int(m2.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base, recs, tot = None, [], 0.0
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    base = a if base is None else base
    a -= base
    s = float(r[iss] or 0)
    tot += s
    ln = addr_line.get(a)
    if ln and phase_of(ln[0]) == want:
        recs.append((s, a, r[isrc].strip(), ln, {hdr[i][6:]: float(r[i] or 0) for i in sc}))
print(f"{want}: {100 * sum(x[0] for x in recs) / tot:.1f}% of samples")
for s, a, t, ln, d in sorted(recs, reverse=True)[:top]:
    topr = sorted(((v, k) for k, v in d.items() if v > 0), reverse=True)[:2]
    print(f"{100 * s / tot:5.2f}% {a:6x} L{ln[0]} {str(ln[1])[:18]:18s} {t[:58]:58s} {topr}")
