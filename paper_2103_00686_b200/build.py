"""Build libfae.so in-tree: nvcc for sm_100a, linked against the NCCL that
torch bundles (so one NCCL is loaded per process)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libfae.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    try:
        import nvidia.nccl as nn
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def cublas_paths():
    try:
        import nvidia.cublas as nc
        base = list(nc.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "cublas_v2.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/local/cuda/include", "/usr/local/cuda/lib64"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        [os.path.join(ROOT, "include", "fae.h")]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(f) > t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, defines=(), out: str = OUT) -> str:
    """Compile every csrc/*.cu to an object in parallel (one nvcc per file),
    then link libfae.so (`defines`/`out`: an A/B variant build)."""
    if not force and out == OUT and not stale():
        return OUT
    os.makedirs(os.path.dirname(out), exist_ok=True)
    inc, lib = nccl_paths()
    binc, blib = cublas_paths()
    objdir = os.path.join(HERE, "_lib", "obj" + ("_" + os.path.basename(out)[:-3] if out != OUT else ""))
    os.makedirs(objdir, exist_ok=True)
    common = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
              "-I", inc, "-I", binc, "-I", os.path.join(ROOT, "include"), *["-D" + d for d in defines]]
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        procs.append((src, subprocess.Popen(common + ["-c", src, "-o", obj],
                                            stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
    failed = False
    for src, pr in procs:
        so, err = pr.communicate()
        if pr.returncode != 0:
            failed = True
            sys.stderr.write(so + err)
        elif verbose:
            sys.stderr.write(err)
    if failed:
        raise RuntimeError("nvcc failed building libfae.so")
    cmd = ["nvcc", *ARCH, "-shared", "-o", out + ".tmp", *objs,
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath," + lib,
           "-L", blib, "-l:libcublas.so.12", "-l:libcublasLt.so.12", "-Xlinker", "-rpath," + blib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libfae.so")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=os.path.abspath(outs[0]) if outs else OUT))
