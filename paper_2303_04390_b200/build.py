"""Build the native library in-tree (sm_100a only).

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared ...
        -> paper_2303_04390_b200/lib/libphylograd.so
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIB_DIR, "libphylograd.so")
SOURCES = ["phylograd.cu", "schedule.cpp"]
# measurement helper for bench.py (FP64 peak probe; not the hot path, not the ABI)
PROBE = os.path.join(LIB_DIR, "libpgprobe.so")
PROBE_SOURCES = ["probe.cu"]
HEADER_GLOBS = ("*.cuh", "*.hpp", "*.h")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def _inputs():
    import glob
    files = [os.path.join(CSRC, f) for f in SOURCES]
    for g in HEADER_GLOBS:
        files += glob.glob(os.path.join(CSRC, g))
    files.append(os.path.join(os.path.dirname(HERE), "include", "phylograd.h"))
    files.append(os.path.abspath(__file__))
    return files


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(PROBE):
        return True
    t = min(os.path.getmtime(LIB), os.path.getmtime(PROBE))
    return any(os.path.getmtime(f) > t for f in _inputs() + [os.path.join(CSRC, f) for f in PROBE_SOURCES])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB, *[os.path.join(CSRC, f) for f in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    probe = [nvcc, *NVCC_FLAGS, "-o", PROBE, *[os.path.join(CSRC, f) for f in PROBE_SOURCES]]
    procs = [subprocess.Popen(c) for c in (cmd, probe)]
    for p, c in zip(procs, (cmd, probe)):
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, c)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
