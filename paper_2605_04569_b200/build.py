"""Build the in-tree sm_100a shared library `libisa_b200.so` with nvcc.

    python -m paper_2605_04569_b200.build          # or __graft_entry__.build()

The library is plain C ABI (include/isa_b200.h); Python binds it with ctypes
(paper_2605_04569_b200/_native.py). No torch extension machinery is used, so
the .so has no torch types in its signatures and travels with the repo
snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libisa_b200.so")
SOURCES = ["isa_capi.cu"]
DEPS = ["isa_capi.cu", "isa_attn.cuh", "isa_route.cuh", "isa_ptx.cuh", "isa_bwd.cuh", "isa_bwd_tc.cuh", "isa_taylor_t.cuh"]


def nvcc_path() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build libisa_b200.so")
    return cand


def nvcc_command(out: str = LIB) -> list[str]:
    return [
        nvcc_path(),
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC", "-shared",
        "-Xptxas", "-v",
        "-I", os.path.join(ROOT, "include"),
        *(["-DISA_DEBUG_WAIT"] if os.environ.get("ISA_DEBUG_WAIT") else []),
        *([f"-D{f}" for f in os.environ.get("ISA_EXTRA_DEFINES", "").split(",") if f]),
        "-o", out,
        *[os.path.join(CSRC, s) for s in SOURCES],
    ]


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    files = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "isa_b200.h")]
    return any(os.path.getmtime(f) > t for f in files if os.path.exists(f))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not is_stale():
        return LIB
    cmd = nvcc_command()
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    with open(os.path.join(HERE, "build.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{log[-4000:]}")
    if "spill" in log:
        spills = [l for l in log.splitlines() if "spill" in l and not l.strip().startswith("0 bytes")]
        bad = [l for l in spills if " 0 bytes spill stores, 0 bytes spill loads" not in l]
        if bad and verbose:
            print("\n".join(bad), file=sys.stderr)
    if verbose:
        print(log[-2000:])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
