"""Build libavion_b200.so in-tree: nvcc, sm_100a only, C ABI (include/avion_b200.h).

    python -m paper_2309_16669_b200.build          # incremental
    python -m paper_2309_16669_b200.build --clean

Objects go to build/, the library to paper_2309_16669_b200/libavion_b200.so
(git-ignored, but shipped to the GPU box by gpurun).
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD_ROOT = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libavion_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
          "-Xptxas", "-v" if os.environ.get("AVB_PTXAS_VERBOSE") else "-O3",
          "-I" + os.path.join(ROOT, "include")] + os.environ.get("AVB_NVCC_DEFS", "").split()
# AVB_NVCC_DEFS: extra defines for debug builds, e.g. "-DAVB_ATTN_TRACE_HOOKS" or "-DAVB_DEBUG_KNOBS".
# Objects live in a directory keyed by a hash of every flag, so a debug build never leaks into a
# product build (the library itself is always relinked when the flag set changes).
_FLAG_KEY = hashlib.sha1(" ".join([NVCC, *ARCH, *CFLAGS]).encode()).hexdigest()[:12]
BUILD = os.path.join(BUILD_ROOT, "avion-" + _FLAG_KEY)
STAMP = LIB + ".flags"


def _deps(src: str) -> list[str]:
    return [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "avion_b200.h")]


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    if _stale(obj, _deps(src)):
        cmd = [NVCC, *ARCH, *CFLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}\n{r.stdout}")
        return obj, r.stderr
    return obj, ""


def build(clean: bool = False, verbose: bool = False) -> str:
    if clean and os.path.isdir(BUILD):
        shutil.rmtree(BUILD)
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, srcs))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    stamp_ok = os.path.exists(STAMP) and open(STAMP).read().strip() == _FLAG_KEY
    if _stale(LIB, objs) or not stamp_ok:
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
        with open(STAMP, "w") as fh:
            fh.write(_FLAG_KEY + "\n")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.clean, a.verbose))
