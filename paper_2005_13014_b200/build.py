"""Build liboec.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2005_13014_b200.build [--force] [--verbose]

--fmad=false is part of the PRODUCT build, not a debug switch: the kernels are HBM-bound, so FMA
contraction buys no speed, and keeping every + - * / separately rounded in the definition's order
makes the GPU results bit-identical to the CPU oracle (R3, R13).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liboec.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3",
    "-lineinfo",
    "--fmad=false",
    "-std=c++17",
    "-shared",
    "-Xcompiler",
    "-fPIC,-O2,-ffp-contract=off",
    "-I" + os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "oec.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """defines: extra -D tile parameters (HD_V, HD_JB, HD_S, HD_NW, VA_NC, VA_LB, VA_S) for tuning
    builds written to `out`; the product build uses the defaults in the sources."""
    if not force and out == LIB and not defines and not _stale():
        return LIB
    # one nvcc per translation unit in parallel (no device code crosses TUs), then one link
    from concurrent.futures import ThreadPoolExecutor

    cflags = [f for f in FLAGS if f != "-shared"]
    objdir = out + ".objs"
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *cflags, *(["-Xptxas", "-v"] if verbose else []), *["-D" + d for d in defines], "-c", src,
               "-o", obj]
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(compile_one, sources()))
    subprocess.check_call([NVCC, *ARCH, "-shared", *objs, "-o", out + ".tmp", "-ldl"])
    os.replace(out + ".tmp", out)
    for o in objs:
        os.remove(o)
    os.rmdir(objdir)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, defines=defs, out=outs[0] if outs else LIB))
