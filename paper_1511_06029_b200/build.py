"""Build libqtt_b200.so in-tree with nvcc for sm_100a (no JIT cache).

    python -m paper_1511_06029_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.environ.get("QTT_OBJ_DIR", os.path.join(PKG, "build"))
LIB = os.environ.get("QTT_LIB_OUT", os.path.join(PKG, "libqtt_b200.so"))

SOURCES = ["qtt_dmma_inst_kb12.cu", "qtt_dmma_inst_kb34.cu", "qtt_dmma_inst_kb56.cu", "qtt_dmma_inst_kb78.cu",
           "qtt_wide_kernel.cu", "qtt_morton.cu", "qtt_compressed.cu", "qtt_level_dmma.cu",
           "qtt_plan.cpp", "qtt_runtime.cpp", "qtt_host_copy.cpp", "qtt_api.cpp", "qtt_api_ext.cpp"]
HEADERS = ["qtt_internal.h", "qtt_runtime.h", "qtt_dmma_kernel.cuh", os.path.join("..", "..", "include", "qtt.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                  "-I" + os.path.join(ROOT, "include")]
# experiment knobs (A/B builds): QTT_EXTRA_NVFLAGS="-DQTT_CG3_MIN_NB=6" QTT_LIB_OUT=path
NVFLAGS += os.environ.get("QTT_EXTRA_NVFLAGS", "").split()


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _newest_input() -> float:
    paths = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    paths.append(os.path.abspath(__file__))
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str) -> str:
    os.makedirs(OBJ, exist_ok=True)
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    cmd = [nvcc()] + NVFLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cu"):
        cmd[1:1] = ["-Xptxas", "-v"] if os.environ.get("QTT_PTXAS_V") else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_input():
        return LIB
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", LIB + ".tmp"] + objs
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
