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
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d, indent=1))
