"""In-tree build of libtofu.so (sm_100a).  Used by __graft_entry__.build().

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo, static cudart, no torch types.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libtofu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    cu = sorted(glob.glob(os.path.join(PKG, "csrc", "cuda", "*.cu")))
    cpp = sorted(glob.glob(os.path.join(PKG, "csrc", "host", "*.cpp")))
    return cu, cpp


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = True) -> str:
    cu, cpp = sources()
    hdrs = glob.glob(os.path.join(PKG, "csrc", "**", "*.h*"), recursive=True) + [os.path.join(ROOT, "include", "tofu.h")]
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest(cu + cpp + hdrs):
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
             "-I", os.path.join(PKG, "csrc")]
    objs = []
    procs = []
    for src in cu + cpp:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _newest(hdrs)):
            continue
        cmd = [NVCC] + ARCH + flags + ["-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC] + flags + ["-x", "c++", "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"compile failed: {' '.join(cmd)}")
    link = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl", "-lpthread", "-lrt"]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(r.stdout.decode())
        raise RuntimeError("link failed")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
