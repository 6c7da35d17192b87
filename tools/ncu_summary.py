"""Summarise an ncu report: key metrics, stall reasons, SASS opcode mix."""
import csv
import subprocess
import sys
from collections import Counter


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2]))


def sass(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[1], rows[2:]


def main(rep, top=18):
    d = raw(rep)
    keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
            "smsp__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.per_cycle_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "dram__bytes_read.sum", "dram__bytes_write.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]
    for k in keys:
        print(f"{k:70s} {d.get(k)}")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("stalls:", ", ".join(f"{k} {100*v/tot:.1f}%" for v, k in sorted(st, reverse=True)[:10]))
    hdr, data = sass(rep)
    iS, iE, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
    cs, ce = Counter(), Counter()
    for r in data:
        toks = r[iSrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        cs[op] += float(r[iS] or 0)
        ce[op] += float(r[iE] or 0)
    ts, te = sum(cs.values()) or 1, sum(ce.values()) or 1
    print("opcodes (instr%, stall%):", ", ".join(f"{op} {100*ce[op]/te:.1f}/{100*cs[op]/ts:.1f}"
                                                 for op, _ in ce.most_common(top)))


if __name__ == "__main__":
    main(sys.argv[1])
