"""Key metrics of the persistent kernel from one `ncu --set full` capture, as the
JSON bench.py reads for roofline.traffic / fp64 pipe activity.
Usage: ncu_json.py REP CONFIG PRECISION OUT.json"""
import csv
import json
import subprocess
import sys

rep, config, precision, out = sys.argv[1:5]
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1.0, "us": 1e-3, "ns": 1e-6,
         "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6}


def get(k, scale=True):
    i = hdr.index(k)
    v = float(vals[i].replace(",", ""))
    return v * SCALE.get(units[i], 1.0) if scale else v


d = {
    "config": config, "precision": precision, "report": rep.split("/")[-1],
    "kernel": vals[hdr.index("Kernel Name")],
    "duration_ms": get("gpu__time_duration.sum"),
    "dram_read_bytes": get("dram__bytes_read.sum"),
    "dram_write_bytes": get("dram__bytes_write.sum"),
    "fp64_pipe_active_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", False),
    "issue_active_per_cycle": get("smsp__issue_active.avg.per_cycle_active", False),
    "warps_active_per_cycle": get("smsp__warps_active.avg.per_cycle_active", False),
    "registers_per_thread": get("launch__registers_per_thread", False),
    "grid": get("launch__grid_size", False), "block": get("launch__block_size", False),
    "inst_executed": get("smsp__inst_executed.sum", False),
}


def opt(k):
    return get(k, False) if k in hdr else None


# executed fp64 work, per elapsed cycle over the whole GPU (thread-level SASS
# counts; clock independent): the fraction of the DFMA lanes' peak the kernel
# keeps busy (slots: one DFMA, DMUL or DADD each) and its flop-weighted twin
# (a DFMA is 2 flops; peak = 2 x 64 DFMA lanes x SMs per cycle)
ops = {op: opt(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
       for op in ("dfma", "dmul", "dadd")}
peak = opt("sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained")
if all(v is not None for v in ops.values()) and peak:
    d["fp64_thread_ops_per_cycle"] = ops
    d["fp64_peak_thread_ops_per_cycle"] = peak
    d["fp64_slot_frac_executed"] = (ops["dfma"] + ops["dmul"] + ops["dadd"]) / peak
    d["fp64_flop_frac_executed"] = (2 * ops["dfma"] + ops["dmul"] + ops["dadd"]) / (2 * peak)
for k in ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
          "smsp__pcsamp_warps_issue_stalled_long_scoreboard"):
    v = opt(k)
    if v is not None:
        d[k] = v
if len(sys.argv) > 5:
    d["note"] = sys.argv[5]
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d, indent=1))
