"""Build libscpl.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo).

    python -m paper_1903_03180_b200.build_ext [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libscpl.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# (source, object, extra flags): the carve TU is compiled once per DP window width (kc6, kc4, kc3)
SOURCES = [("scpl_energy.cu", "scpl_energy.o", []), ("scpl_stats.cu", "scpl_stats.o", []),
           ("scpl_carve2.cu", "scpl_carve2.o", ["-DSCPL_KC=6"]),
           ("scpl_carve2.cu", "scpl_carve2_kc4.o", ["-DSCPL_KC=4"]),
           ("scpl_carve2.cu", "scpl_carve2_kc3.o", ["-DSCPL_KC=3"]),
           ("scpl_replay.cu", "scpl_replay.o", []), ("scpl_tables.cu", "scpl_tables.o", []),
           ("scpl_api.cu", "scpl_api.o", [])]
HEADERS = ["scpl_common.cuh", "scpl_kernels.h", os.path.join("..", "..", "include", "scpl.h")]
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
    "-fmad=false",          # every fp64 +,* rounds on its own unless written as __fma_rn
    "-Xptxas", "-v",
] + os.environ.get("SCPL_EXTRA_NVCC_FLAGS", "").split()  # experiments only


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def _compile(entry, force: bool) -> str:
    src, objname, extra = entry
    obj = os.path.join(BUILD, objname)
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= _newest(deps):
        return obj
    cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(r.stderr)
    return obj


LIB_CHECKED = os.path.join(HERE, "libscpl_checked.so")  # device invariant checks (SCPL_CHECKED=1)


def _link(lib, objs, force):
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < _newest(objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
               "-o", lib, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")


def build(force: bool = False, checked: bool = True) -> str:
    os.makedirs(BUILD, exist_ok=True)
    entries = [(s, o, e) for s, o, e in SOURCES]
    if checked:  # the same sources with -DSCPL_CHECKS into *_chk.o
        entries += [(s, o.replace(".o", "_chk.o"), e + ["-DSCPL_CHECKS"]) for s, o, e in SOURCES]
    with ThreadPoolExecutor(max_workers=len(entries)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), entries))
    _link(LIB, objs[:len(SOURCES)], force)
    if checked:
        _link(LIB_CHECKED, objs[len(SOURCES):], force)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
