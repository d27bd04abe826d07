"""Build libks_b200.so in-tree: nvcc -gencode arch=compute_100a,code=sm_100a (B200 only).

    python -m paper_1312_1869_b200.build          # incremental
    python -m paper_1312_1869_b200.build --force
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libks_b200.so")
SOURCES = ["ks_api.cu", "ks_sketch.cu", "ks_gauss.cu", "ks_tsqr.cu", "ks_solve.cu", "ks_gp.cu"]
HEADERS = ["ks_common.cuh", "ks_internal.h", "ks_tc.cuh", "ks_tsqr_tc.inc", os.path.join("..", "..", "include", "ks.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v", "-cudart", "static"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    if force or _stale(obj, deps):
        log = obj + ".ptxas.log"
        with open(log, "w") as f:
            subprocess.check_call([NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj], stdout=f, stderr=subprocess.STDOUT)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), SOURCES))
    if force or _stale(LIB, objs):
        subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
                               "-o", LIB, *objs])
        if verbose:
            print(f"built {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
