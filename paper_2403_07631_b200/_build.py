"""Build recipe for libpct.so (sm_100a) — invoked by __graft_entry__.build().

Compiles paper_2403_07631_b200/csrc/*.cu with nvcc into
paper_2403_07631_b200/lib/libpct.so (in-tree, so the .so travels to the GPU box
with the gpurun snapshot).  --fmad=false keeps every float expression
uncontracted (bit-exactness); the Markstein divisions
use explicit fma().  Also builds lib/libpct_hostmath.so: the __host__ side of
csrc/cellmath.cuh for the CPU tests of the per-cell arithmetic.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xptxas", "-v",
              "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-I", str(INCLUDE)]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, sources) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build(force: bool = False, verbose: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    cu = sorted(CSRC.glob("*.cu"))
    # host-only C++ of libpct.so (g++; hostmath.cpp builds libpct_hostmath.so)
    cpp = [p for p in sorted(CSRC.glob("*.cpp")) if p.name != "hostmath.cpp"]
    deps = cu + cpp + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [INCLUDE / "pct.h"]
    out = LIB / "libpct.so"
    if force or _stale(out, deps):
        from concurrent.futures import ThreadPoolExecutor

        def compile_one(src):
            obj = LIB / (src.stem + ".o")
            cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src.name}")
            if verbose:
                sys.stderr.write(r.stderr)
            (LIB / (src.stem + ".ptxas.txt")).write_text(r.stderr)
            return str(obj)

        def compile_cpp(src):
            obj = LIB / (src.stem + ".o")
            cxx = shutil.which("g++") or "g++"
            cmd = [cxx, "-O3", "-std=c++17", "-fPIC", "-pthread", "-I", str(INCLUDE), "-c",
                   str(src), "-o", str(obj)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"g++ failed on {src.name}")
            return str(obj)

        # one compiler per translation unit, in parallel (k_evaluate.cu dominates)
        with ThreadPoolExecutor(max(1, min(len(cu) + len(cpp), os.cpu_count() or 1))) as ex:
            objs = list(ex.map(compile_one, cu)) + list(ex.map(compile_cpp, cpp))
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(out), *objs, "-lcudart", "-Xcompiler",
               "-pthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    host = LIB / "libpct_hostmath.so"
    hsrc = CSRC / "hostmath.cpp"
    if force or _stale(host, [hsrc, CSRC / "cellmath.cuh"]):
        cxx = shutil.which("g++") or "g++"
        cmd = [cxx, "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
               "-I", str(CSRC), str(hsrc), "-o", str(host), "-lm"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("g++ failed on hostmath.cpp")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
