"""Builds the engine's shared library in-tree with nvcc for sm_100a.

Output: paper_2501_06647_b200/_lib/libtucktree_b200.so (git-ignored, travels to
the GPU box with the repo snapshot). Cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libtucktree_b200.so")
SOURCES = ["tt_leaf.cu", "tt_wide.cu", "tt_grid.cu", "tt_grid_solve.cu", "tt_stitch.cu", "tt_stitch_wide.cu", "tt_host.cpp"]
HEADERS = ["tt_common.h", "tt_block.cuh", "tt_dev.cuh", "tt_stitch_body.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    extra = ["-DTT_INSTRUMENT"] if os.environ.get("TT_INSTRUMENT") == "1" else []
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", *extra,
              "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include")]
    # one translation unit per kernel family, compiled in parallel, then linked
    # (objects are kept, so a change to one source recompiles only that unit;
    # a header change recompiles everything)
    objs, procs = [], []
    hdr_t = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)  # (flag changes: the .flags tag)
    api_t = os.path.getmtime(os.path.join(ROOT, "include", "tucktree_b200.h"))  # included by tt_host.cpp only
    tag = os.path.join(OUT_DIR, ".flags")
    flags = " ".join(common)
    if not os.path.exists(tag) or open(tag).read() != flags:
        force = True
    for src in SOURCES:
        obj = os.path.join(OUT_DIR, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(hdr_t, os.path.getmtime(os.path.join(CSRC, src)),
                                                api_t if src == "tt_host.cpp" else 0)):
            continue
        procs.append(subprocess.Popen(common + ["-c", os.path.join(CSRC, src), "-o", obj],
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    if not procs and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(o) for o in objs):
        return LIB  # nothing changed
    errs = []
    for pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            errs.append(out + err)
        elif verbose:
            sys.stderr.write(err)
    if errs:
        sys.stderr.write("\n".join(errs))
        raise RuntimeError("nvcc failed building libtucktree_b200.so")
    r = subprocess.run([NVCC, *ARCH, "-shared", *objs, "-o", LIB + ".tmp"], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libtucktree_b200.so")
    os.replace(LIB + ".tmp", LIB)
    with open(tag, "w") as f:
        f.write(flags)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
