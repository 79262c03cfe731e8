"""Build the in-tree C-ABI library libeagercoll_b200.so for sm_100a.

    python -m paper_1908_04207_b200.build            # or __graft_entry__.build()

nvcc cross-compiles here without a GPU.  The .so lands in
paper_1908_04207_b200/lib/ (git-ignored, shipped to the GPU box by gpurun).
No -use_fast_math and explicit _rn intrinsics: the fixed-order path must stay
bit-exact.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIB_DIR, "libeagercoll_b200.so")
# the checked build: device assertions on ring indices, chunk ranges, slot
# offsets and protocol invariants (EC_ASSERT in csrc/ec_common.cuh); selected
# at import with EC_DEBUG_LIB=1 -- the bounds/race tooling while
# compute-sanitizer is unavailable
LIB_DEBUG = os.path.join(LIB_DIR, "libeagercoll_b200_debug.so")
SOURCES = ["ec_kernels.cu", "ec_host.cu"]
HEADERS = ["ec_common.cuh", "ec_ops.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "eagercoll_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    lib = LIB_DEBUG if debug else LIB
    if not force and not _stale(lib):
        return lib
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, *FLAGS, *(["-DEC_DEBUG"] if debug else []), "-shared", "-o", tmp,
           *[os.path.join(CSRC, f) for f in SOURCES], "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(LIB_DIR, "build_debug.log" if debug else "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    if verbose:
        sys.stdout.write(res.stdout + res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
