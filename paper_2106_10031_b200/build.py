"""Build the in-tree CUDA library _lib/libam_b200.so for sm_100a with nvcc.

The face solver is compiled with -fmad=false so its tolerance decisions use
separately rounded multiply/add (the same arithmetic as the CPU oracle and
numpy); the composition GEMM keeps FMA (it runs on the DMMA pipe anyway).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.environ.get("AM_BUILD_OUT") or os.path.join(HERE, "_lib", "libam_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=default"]
SOURCES = {
    "am_compose.cu": [],
    "am_narrow.cu": [],
    "am_hash.cu": [],
    "am_seed.cu": [],
    "am_engine.cu": [],
    "am_face.cu": ["-fmad=false"],
    "am_peak.cu": [],
    "am_weld.cu": [],
    "am_result.cu": [],
    "am_diag.cu": ["-fmad=false"],
    "am_shard.cu": [],
    "am_trace.cu": ["-fmad=false"],
}


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False) -> str:
    """AM_BUILD_FLAGS (space-separated) are appended to every nvcc compile (e.g. -DAM_FACE_STATS)."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "am_internal.h"), os.path.join(CSRC, "am_ptx.cuh"), os.path.join(CSRC, "am_near.cuh"),
                   os.path.join(os.path.dirname(HERE), "include", "am_b200.h")]
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(d) for d in deps):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    objdir = os.path.join(os.path.dirname(OUT), "obj" if "AM_BUILD_OUT" not in os.environ
                          else "obj_" + os.path.basename(OUT).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for name, extra in SOURCES.items():
        obj = os.path.join(objdir, name.replace(".cu", ".o"))
        cmd = ([nvcc()] + ARCH + COMMON + extra + os.environ.get("AM_BUILD_FLAGS", "").split()
               + ["-c", os.path.join(CSRC, name), "-o", obj])
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    cmd = [nvcc()] + ARCH + ["-shared", "-o", OUT] + objs
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
