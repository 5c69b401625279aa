"""Build the sm_100a shared library in-tree (no JIT cache, travels with the repo).

    python -m paper_1811_11992_b200.build [--verbose]

One translation unit (csrc/capi.cu includes the kernel files), fp64,
``--fmad=false`` so the assembly arithmetic follows the reference's unfused
operation order, ``-lineinfo`` so ncu's source page maps to our code.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIB_DIR, "libiscgpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
         "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh")))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(HERE, "..", "include", "iscgpu.h"), __file__]
    return all(os.path.getmtime(s) <= t for s in deps if os.path.exists(s))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    extra = os.environ.get("ISC_NVCC_EXTRA", "").split()   # experiments, e.g. -DMC_MINB=6
    flags = list(FLAGS)
    if os.environ.get("ISC_FMAD") == "1":   # experiment: contracted a*b+c (not the reference's order)
        flags[flags.index("--fmad=false")] = "--fmad=true"
    cmd = [NVCC, *flags, *extra, "-Xptxas", "-v", "-o", LIB + ".tmp", os.path.join(CSRC, "capi.cu")]
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        errs = [ln for ln in res.stderr.splitlines() if "error" in ln.lower()]
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs[:40]) + "\n" + res.stderr[-3000:])
    os.replace(LIB + ".tmp", LIB)
    with open(os.path.join(LIB_DIR, "ptxas.log"), "w") as fh:
        fh.write(res.stderr)
    if verbose:
        print(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv))
