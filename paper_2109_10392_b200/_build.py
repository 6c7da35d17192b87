"""In-tree build of the sm_100a shared library (``_lib/libbatchmpc_b200.so``).

Plain nvcc, no torch extension machinery: the library exposes only the C ABI
declared in ``include/batchmpc_b200.h`` and is loaded with ctypes.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libbatchmpc_b200.so"
OBJDIR = ROOT / "build" / "obj"
# BMPC_VARIANT=prof builds the phase-profiling library (tools/phase_prof.py)
# next to the product one; it is never loaded by the package itself.
VARIANTS = {"prof": ["-DBMPC_PHASE_PROF"]}

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
# ops.cu restates the reference's scalar C: no FMA contraction there.
UNITS = [
    ("am_solve.cu", "am_solve", []),
    ("ops.cu", "ops", ["-fmad=false"]),
    ("capi.cu", "capi", []),
    ("peak.cu", "peak", []),
    ("steps.cu", "steps", []),
] + [("am_inst.cu", f"am_inst_nb{nb}", [f"-DBMPC_INST_NB={nb}"]) for nb in range(4, 17)]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _stale(out: Path, deps: list[Path]) -> bool:
    return not out.exists() or any(d.stat().st_mtime > out.stat().st_mtime for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str | None = None) -> Path:
    variant = variant if variant is not None else os.environ.get("BMPC_VARIANT", "")
    vflags = (VARIANTS.get(variant, []) + os.environ.get("BMPC_VARIANT_FLAGS", "").split()) if variant else []
    lib = LIB.with_name(f"libbatchmpc_b200_{variant}.so") if variant else LIB
    objdir = OBJDIR.with_name(f"obj_{variant}") if variant else OBJDIR
    LIBDIR.mkdir(parents=True, exist_ok=True)
    objdir.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "batchmpc_b200.h"]
    from concurrent.futures import ThreadPoolExecutor

    jobs, objs = [], []
    for src, name, extra in UNITS:
        s = CSRC / src
        o = objdir / (name + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers]):
            jobs.append(([nvcc(), *ARCH, *COMMON, *vflags, *extra, "-c", str(s), "-o", str(o)], name))

    def run(job):
        cmd, name = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        (objdir / (name + ".ptxas.log")).write_text(r.stdout + r.stderr)
        return name, r

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for name, r in ex.map(run, jobs):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {name}")
            if verbose:
                sys.stderr.write(r.stderr)
    if force or _stale(lib, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(lib), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
