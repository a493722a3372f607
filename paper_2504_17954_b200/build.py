"""Build the in-tree CUDA library ``libivrgs.so`` (sm_100a) with nvcc.

    python -m paper_2504_17954_b200.build [--verbose]

The library exports the C ABI declared in ``include/ivrgs.h``.  It is built
in-tree so the snapshot shipped to the GPU box carries it.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libivrgs.so")
SOURCES = ["abi.cu", "preprocess.cu", "sort.cu", "blend.cu", "backward.cu", "vq.cu", "sh.cu", "ivrg.cu", "ssim.cu", "regularize.cu", "adam.cu", "concat.cu", "display.cu", "dvr.cu", "trainstep.cu", "inverse.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# Translation units whose float64 chains must reproduce numpy's rounding op by
# op (K1 preprocess, K8 SH colour, K10 pseudo normals): no FMA contraction.
# Everywhere else the reference-exact steps use the explicitly rounded
# intrinsics of ivr_common.cuh (dmul/dadd/...), so the rest of the code may
# contract a*b+c into FMAs.
EXACT_TUS = {"preprocess.cu", "sh.cu", "regularize.cu"}


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(REPO, "include", "ivrgs.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False):
    if not force and not needs_build():
        return LIB
    objdir = os.path.join(PKG, "_obj")
    os.makedirs(objdir, exist_ok=True)
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-I" + os.path.join(REPO, "include"), "--expt-relaxed-constexpr"]
    if verbose:
        flags += ["-Xptxas", "-v"]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        fmad = "-fmad=false" if os.path.basename(src) in EXACT_TUS else "-fmad=true"
        procs.append((src, subprocess.Popen([nvcc(), *flags, fmad, "-c", src, "-o", obj],
                                            stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(out.decode())
        if p.returncode:
            failed = True
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = LIB + ".tmp"
    subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force=True)
    print(LIB)
