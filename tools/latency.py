"""Print dependent-chain latencies (SM cycles/op) measured on the device."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2109_10392_b200 import _native as nat  # noqa: E402

torch.cuda.init()
names = ["DFMA", "DADD", "DMUL", "MUFU.RSQ64H", "FFMA", "LDS.64 chase", "SHFL.64", "rsqrt_nb"]
lib = nat.load()
for i, nm in enumerate(names):
    v = ctypes.c_double()
    nat.check(lib.bmpc_latency_probe(i, ctypes.byref(v), None))
    print(f"{nm:14s} {v.value:6.2f} cycles")
