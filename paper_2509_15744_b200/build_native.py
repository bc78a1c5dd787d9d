"""Build the in-tree native library libwaveb200.so for sm_100a.

    python -m paper_2509_15744_b200.build_native

The library links csrc/capi.cu (C ABI, aux kernels) with the per-dtype
step-engine units csrc/step_*.cu and csrc/step2_*.cu, compiled in parallel.  Flags: -fmad=false -prec-div=true -ftz=false keep every field
operation a single IEEE round-to-nearest op in source order, which is what
makes the fp64 AND fp32 builds bit-exact against the reference
(DESIGN.md "Arithmetic contract").
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libwaveb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "--cudart", "static", "-lpthread"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh")))


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(HERE, "..", "include", "waveb200.h"), __file__]
    return all(os.path.getmtime(p) <= t for p in deps if os.path.exists(p))


def build(force=False, verbose=False, extra=(), out=None):
    lib = out or LIB
    if out is None and not force and up_to_date():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    units = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    tag = os.path.basename(lib).replace(".", "_")
    objs = [os.path.join(OUT_DIR, f"{tag}_{u[:-3]}.o") for u in units]
    cmds = [[NVCC, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, u), "-o", o]
            for u, o in zip(units, objs)]
    if verbose:
        for c in cmds:
            print(" ".join(c))
    procs = [subprocess.Popen(c) for c in cmds]
    rcs = [p.wait() for p in procs]
    if any(rcs):
        raise subprocess.CalledProcessError(max(rcs), cmds[rcs.index(max(rcs))])
    link = [NVCC, *LINK_FLAGS, *objs, "-o", lib + ".tmp"]
    if verbose:
        print(" ".join(link))
    subprocess.run(link, check=True)
    os.replace(lib + ".tmp", lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    # --force, --ptxas, -DNAME=VALUE (kernel variants), --out=PATH (variant library)
    args = sys.argv[1:]
    extra = [a for a in args if a.startswith("-D")]
    if "--ptxas" in args:
        extra += ["-Xptxas", "-v"]
    outs = [a.split("=", 1)[1] for a in args if a.startswith("--out=")]
    print(build(force="--force" in args, verbose=True, extra=extra,
                out=os.path.abspath(outs[0]) if outs else None))
