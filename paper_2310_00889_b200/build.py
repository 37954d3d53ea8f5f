"""Build libslb.so (hand-written CUDA for sm_100a) in-tree with nvcc.

Each translation unit is compiled to an object in parallel (build/obj/), then linked into the
shared library; a unit is recompiled only when it, a csrc header or include/slb.h changed."""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SO = os.path.join(PKG, "libslb.so")
OBJ = os.path.join(PKG, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=default", "-I", os.path.join(ROOT, "include")]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cpp")))


def _headers():
    return (glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + glob.glob(os.path.join(PKG, "csrc", "*.inc")) +
            [os.path.join(ROOT, "include", "slb.h")])


def _obj(src):
    return os.path.join(OBJ, os.path.basename(src) + ".o")


def stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in sources() + _headers())


def _compile(src, verbose):
    cmd = [NVCC, *FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-c", "-o", _obj(src), src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, r


def build(force=False, verbose=False):
    if not force and not stale():
        return SO
    os.makedirs(OBJ, exist_ok=True)
    th = max([os.path.getmtime(h) for h in _headers()])
    todo = [s for s in sources()
            if force or not os.path.exists(_obj(s)) or os.path.getmtime(_obj(s)) < max(th, os.path.getmtime(s))]
    with cf.ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4) or 1) as ex:
        for src, r in ex.map(lambda s: _compile(s, verbose), todo):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed compiling {os.path.basename(src)}")
            if verbose:
                sys.stderr.write(r.stderr)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", SO,
           *[_obj(s) for s in sources()], "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libslb.so")
    return SO


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(SO)
