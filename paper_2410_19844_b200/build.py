"""Build the in-tree CUDA library libsos_b200.so for sm_100a with nvcc."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsos_b200.so")
# experiment build (-DSOS_EXPERIMENTS): the environment switches and probes of
# DESIGN.md 5.4; never loaded by the package unless a tool asks for it
LIB_EXP = os.path.join(HERE, "libsos_b200_exp.so")
SOURCES = ["sos_api.cu", "sos_index.cu", "sos_pointwise.cu", "sos_gemmq.cu", "sos_tiny.cu"]
HEADERS = ["sm100_ptx.cuh", "sos_internal.cuh", "sos_slice.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "sos_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, experiments: bool = False) -> str:
    lib = LIB_EXP if experiments else LIB
    if not force and not _stale(lib):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    extra = ["-DSOS_EXPERIMENTS"] if experiments else []
    cmd = [NVCC, *FLAGS, *extra, "-o", tmp, *[os.path.join(CSRC, f) for f in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    if not experiments:
        with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
            f.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose=True, experiments="--experiments" in sys.argv))
