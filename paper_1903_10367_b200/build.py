"""Build libtmg.so in-tree with nvcc for sm_100a.

    python -m paper_1903_10367_b200.build [--force] [-v]

Two translation units, compiled in parallel and linked into one shared
library:

* ``engine.cu`` (the C ABI and the 2D engine) with ``--fmad=false``: the 2D
  kernels round every product and sum separately, as numpy does, so they
  reproduce the reference's iterates bit for bit;
* ``engine3.cu`` (the 3D engine) with FMA contraction: there is no 3D
  reference, and the north star's bar is relative 1e-10 against the 3D
  oracle, which the contracted kernels meet with margin (tests pin it).

The ptxas resource report goes to ``build/ptxas_report.txt`` (untracked).
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtmg.so")
OBJDIR = os.path.join(ROOT, "build")
REPORT = os.path.join(OBJDIR, "ptxas_report.txt")
UNITS = [("engine.cu", ["--fmad=false"]), ("engine3.cu", ["--fmad=true"])]
DEPS = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "tmg.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    inc = [f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
    procs = []
    for src, extra in UNITS:
        obj = os.path.join(OBJDIR, src.replace(".cu", ".o"))
        cmd = [nvcc(), *NVCC_FLAGS, *extra, *os.environ.get("TMG_NVCC_FLAGS", "").split(), *inc, "-c", "-o", obj,
               os.path.join(CSRC, src)]
        procs.append((obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    report, objs = [], []
    for obj, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + out + err)
        report.append(err)
        objs.append(obj)
    res = subprocess.run([nvcc(), "-shared", "-o", LIB, *objs], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n" + res.stdout + res.stderr)
    if verbose:
        sys.stdout.write("".join(report))
    with open(REPORT, "w") as fh:
        fh.write("".join(report))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
