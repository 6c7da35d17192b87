"""Operator-level tail_core / tail_update timing on device tensors (the kernels
behind the reference's registry back-end).  Usage: tail_timing.py [l ...]
(BMPC_LIB selects the library)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2109_10392_b200 import kernels  # noqa: E402

n, m = 100, 10
for l in [int(a) for a in sys.argv[1:]] or [1024, 16384]:
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=g)  # noqa: E731
    args = (r(n, l) * 50, r(n, l) * 4, r(n, l) * 10 + 20, r(n, l), r(n, l) * 3, r(n, l) * 3, r(n, l) * 0.1,
            r(m * n) * 50, r(m * n) * 4, 0.1, 35.0, 8.0, 5.6, 2.4)
    for name, fn in (("tail_core", kernels.tail_core), ("tail_update", kernels.tail_update)):
        for _ in range(3):
            fn(*args)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            out = fn(*args)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} n={n} m={m} l={l}: {e0.elapsed_time(e1) / 10:.3f} ms per call (allocations included)")
