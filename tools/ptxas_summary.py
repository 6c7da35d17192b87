"""Per-kernel registers / spills from an nvcc -Xptxas -v log: name regs spill_st spill_ld."""
import re
import sys


def parse(path):
    out, cur = {}, None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            k = re.search(r"am_solve_kernelIL(i\d+)ELi(\d+)ELb(\d)ELb(\d)ELb(\d)E(?:Lb(\d)E)?", cur)
            cur = ("am<" + ",".join(g.lstrip("i") for g in k.groups() if g is not None) + ">") if k else cur[:40]
            out[cur] = [None, 0, 0]
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and out[cur][0] is None:
            out[cur][1] += int(m.group(1))
            out[cur][2] += int(m.group(2))
        m = re.search(r"Used (\d+) registers", line)
        if m:
            out[cur][0] = int(m.group(1))
    return out


if __name__ == "__main__":
    logs = [parse(p) for p in sys.argv[1:]]
    for k in logs[0]:
        print(k, *["%s/%s/%s" % tuple(l.get(k, ["-"] * 3)) for l in logs])
