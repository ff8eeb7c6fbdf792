"""Build libisogs.so (the C-ABI CUDA library) in-tree for sm_100a.

    python -m paper_2509_05216_b200.build

Compiles every csrc/*.cu with nvcc for `-gencode arch=compute_100a,
code=sm_100a -lineinfo` and links them into paper_2509_05216_b200/_build/
libisogs.so (static cudart, so the library is self-contained and travels with
the repository snapshot).  Translation units on the float64 key path are built
with -fmad=false (no FMA contraction, like numba).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libisogs.so")
ROOT = os.path.dirname(HERE)

SOURCES = {
    # file: extra flags
    "project.cu": ["-fmad=false"],
    "binning.cu": [],
    "raster_f64.cu": ["-fmad=false"],
    "raster_f32.cu": ["-ftz=true"],
    "loss.cu": [],
    "dist.cu": [],
    "knn.cu": ["-fmad=false"],
    "chain_f32.cu": [],
    "volume.cu": ["-fmad=false"],
    "probe.cu": [],
    "radix.cu": [],
    "api.cu": [],
}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers() -> list[str]:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "isogs.h"))
    return hs


def _compile(src: str, extra: list[str], log: bool) -> str:
    obj = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
    if not _stale(obj, [os.path.join(CSRC, src)] + _headers()):
        return obj
    cmd = [nvcc(), *ARCH, *COMMON, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    with open(obj + ".ptxas.txt", "w") as fh:
        fh.write(res.stderr)
    if log:
        print(f"compiled {src}", file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda kv: _compile(kv[0], kv[1], verbose), SOURCES.items()))
    if _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
        if verbose:
            print(f"linked {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
