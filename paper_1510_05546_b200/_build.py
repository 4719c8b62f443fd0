"""Build libgtcp.so in-tree with nvcc for sm_100a (B200)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "_lib", "libgtcp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dirs():
    import nvidia.nccl  # the NCCL torch links against (same soname, loaded once)
    base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu"))) + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + \
        [os.path.join(ROOT, "include", "gtcp.h")]


def build(force: bool = False, verbose: bool = False, debug: bool = False, defines=(), out: str | None = None) -> str:
    """defines / out: experiment builds (extra -D flags into another .so)."""
    srcs = sources()
    LIB = globals()["LIB"] if not debug else os.path.join(HERE, "_lib", "libgtcp_debug.so")
    if out:
        LIB = out
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(s) for s in srcs):
        return LIB
    inc, lib = nccl_dirs()
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", inc,
           "-o", tmp] + [s for s in srcs if s.endswith(".cu")] + \
          ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib] + \
          (["-DGTCP_DEBUG"] if debug else []) + ["-D" + d for d in defines]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libgtcp.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose="-v" in sys.argv, debug="--debug" in sys.argv,
                defines=defs, out=outs[0] if outs else None))
