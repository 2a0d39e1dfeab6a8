"""Builds libensei_gpu.so IN-TREE with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2003_05328_b200.build        # or __graft_entry__.build()

The .so sits next to this file so it travels to the GPU box with the repo
snapshot; the Python binding (_lib.py) refuses to run without it.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libensei_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-v", "-cudart", "static", "-Wno-deprecated-gpu-targets"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _digest():
    h = hashlib.sha256()
    for d in (CSRC, os.path.join(os.path.dirname(HERE), "include")):
        for root, _, files in os.walk(d):
            for f in sorted(files):
                with open(os.path.join(root, f), "rb") as fh:
                    h.update(f.encode() + fh.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def _obj_digest(src):
    """Per-object key: the source itself, every header it can include, the flags."""
    h = hashlib.sha256()
    with open(src, "rb") as fh:
        h.update(fh.read())
    for d in (CSRC, os.path.join(os.path.dirname(HERE), "include")):
        for root, _, files in os.walk(d):
            for f in sorted(files):
                if not f.endswith(".cu"):
                    with open(os.path.join(root, f), "rb") as fh:
                        h.update(f.encode() + fh.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    stamp = OUT + ".sha"
    dig = _digest()
    if not force and os.path.exists(OUT) and os.path.exists(stamp) and open(stamp).read() == dig:
        return OUT
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        odig = _obj_digest(src)
        ostamp = obj + ".sha"
        if not force and os.path.exists(obj) and os.path.exists(ostamp) and open(ostamp).read() == odig:
            continue  # unchanged translation unit
        cmd = [NVCC, *ARCH, *FLAGS, "-I", os.path.join(os.path.dirname(HERE), "include"), "-dc" if False else "-c",
               src, "-o", obj]
        log = open(obj + ".log", "w")
        procs.append((subprocess.Popen(cmd, stdout=log, stderr=subprocess.STDOUT), src, obj, odig))
    bad = []
    for p, src, obj, odig in procs:
        if p.wait() != 0:
            bad.append(src)
        else:
            with open(obj + ".sha", "w") as f:
                f.write(odig)
    if bad:
        for src in bad:
            sys.stderr.write(open(os.path.join(objdir, os.path.basename(src)[:-3] + ".o.log")).read())
        raise RuntimeError("nvcc failed for: " + ", ".join(bad))
    if verbose:
        for o in objs:
            if not os.path.exists(o + ".log"):
                continue
            sys.stdout.write(open(o + ".log").read())
    link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", OUT, *objs, "-lpthread"]
    subprocess.run(link, check=True)
    with open(stamp, "w") as f:
        f.write(dig)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
