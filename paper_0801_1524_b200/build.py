"""Build libsft.so in-tree with nvcc for sm_100a (no JIT cache, no torch types).

Each source is compiled to an object in parallel (-rdc off, plain -c) and
linked with nvcc -shared; objects are rebuilt when their source, the internal
header or include/sft.h is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libsft.so")
SOURCES = ["api.cu", "tree.cu", "kernels.cu", "translate.cu", "tables.cpp", "comm.cu"]
HEADERS = [os.path.join(CSRC, "sft_internal.cuh"), os.path.join(HERE, "..", "include", "sft.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-O3",
]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _sources():
    return [f for f in SOURCES if os.path.exists(os.path.join(CSRC, f))]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = _mtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + HEADERS
    return any(_mtime(p) > t for p in deps)


def _compile(src, obj, extra, verbose, force):
    path = os.path.join(CSRC, src)
    hdr_t = max(_mtime(h) for h in HEADERS + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")])
    if not force and _mtime(obj) > max(_mtime(path), hdr_t):
        return
    cmd = [NVCC, *FLAGS, *extra, "-c", "-o", obj + ".tmp"]
    cmd += ["-x", "cu", path] if src.endswith(".cpp") else [path]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(obj + ".tmp", obj)


def build(force: bool = False, verbose: bool = False, extra=(), out=None) -> str:
    if out is None and not force and not _stale():
        return LIB
    target = out or LIB
    tag = "" if not extra else "_" + str(abs(hash(tuple(extra))))
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    objs = [os.path.join(OBJ, os.path.splitext(f)[0] + tag + ".o") for f in srcs]
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        list(ex.map(lambda so: _compile(so[0], so[1], list(extra), verbose, force or bool(extra)), zip(srcs, objs)))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", target + ".tmp", *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, extra=["-Xptxas", "-v"] if "-v" in sys.argv else [])
