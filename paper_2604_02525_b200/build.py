"""Build libadahop.so in-tree: nvcc for sm_100a, cudart linked statically.

Usage: python paper_2604_02525_b200/build.py [--verbose]   (run by path: importing the
package itself requires the built library)
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libadahop.so")
SOURCES = ["api.cu", "quant.cu", "quant_tc.cu", "gemm_mxf4.cu", "gemm_mxf4_2sm.cu", "gemm_bf16.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    # bit-exactness contract: IEEE fp32 (no FTZ, no fast math, no FMA contraction in the
    # quantiser path which uses explicit _rn intrinsics anyway)
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-I" + os.path.join(ROOT, "include"),
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "adahop.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), out: str = LIB) -> str:
    if not force and not needs_build():
        return LIB
    objs = []
    bdir = os.path.join(PKG, "build" if out == LIB else "build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *["-D" + d for d in defines], "-Xptxas", "-v" if verbose else "-O3", "-dc" if False else "-c",
               os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        log, _ = p.communicate()
        if verbose or p.returncode != 0:
            sys.stderr.write(f"--- {src}\n{log}")
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    # the exported C ABI symbols are marked default-visible in api.cu via a version script
    ver = os.path.join(bdir, "exports.map")
    with open(ver, "w") as f:
        f.write("{ global: adahop_*; local: *; };\n")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           *objs, "-o", out, "-Xlinker", f"--version-script={ver}", "-lpthread", "-ldl", "-lrt"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError("link failed")
    return out


if __name__ == "__main__":
    # --define NAME=VAL (repeatable) and --out PATH build an experiment variant of the library
    args = sys.argv[1:]
    defs = [args[i + 1] for i, a in enumerate(args) if a == "--define"]
    out = next((args[i + 1] for i, a in enumerate(args) if a == "--out"), LIB)
    print(build(verbose="--verbose" in args, force=True, defines=defs, out=os.path.abspath(out)))
