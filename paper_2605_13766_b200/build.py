"""In-tree build of libelasticarod.so for sm_100a (explicit nvcc; no JIT cache).

    python paper_2605_13766_b200/build.py            # incremental
    python paper_2605_13766_b200/build.py --force
(run by path: importing the package loads the library it builds)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# ER_BUILD_OUT: build a variant library elsewhere (A/B measurements; lib_ab/ is git-ignored)
OUT = os.path.abspath(os.environ.get("ER_BUILD_OUT", os.path.join(HERE, "lib", "libelasticarod.so")))
SOURCES = ["er_api.cu", "er_kernels.cu", "er_warp.cu", "er_contact.cu"]
# per-file flags: the contact narrow phase takes its branch decisions on IEEE-rounded products
# and sums in the order written (no FMA contraction; DESIGN §3 #27)
FILE_FLAGS = {"er_contact.cu": ["-fmad=false"]}
HEADERS = ["er_layout.h", "er_math.cuh", "er_tma.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def _deps():
    return ([os.path.join(CSRC, s) for s in SOURCES + HEADERS]
            + [os.path.join(ROOT, "include", "er.h"), os.path.abspath(__file__)])


def build(force: bool = False, verbose: bool = False) -> str:
    extra = os.environ.get("ER_NVCC_EXTRA", "").split()  # experiments only (e.g. -DER_...)
    stamp = OUT + ".flags"  # the extra flags the library was built with: a change forces a rebuild
    same_flags = os.path.exists(stamp) and open(stamp).read() == " ".join(extra)
    if (not force and same_flags and os.path.exists(OUT)
            and os.path.getmtime(OUT) >= max(os.path.getmtime(p) for p in _deps())):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    objdir = os.path.join(os.path.dirname(OUT), "obj")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:  # the translation units compile concurrently
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *[f for f in FLAGS if f != "-shared"], *FILE_FLAGS.get(src, []), *extra, "-c",
               "-I", os.path.join(ROOT, "include"), "-I", CSRC, os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for src, pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc failed compiling {src}")
        if verbose:
            sys.stderr.write(err)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", OUT + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libelasticarod.so")
    os.replace(OUT + ".tmp", OUT)
    with open(stamp, "w") as f:
        f.write(" ".join(extra))
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
