"""In-tree build of libhprlp_b200.so for sm_100a (nvcc cross-compiles; no GPU needed)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "hpr_capi.cu"), os.path.join(HERE, "csrc", "hpr_mps.cpp")]
DEPS = SRC + [os.path.join(HERE, "csrc", f) for f in sorted(os.listdir(os.path.join(HERE, "csrc")))
              if f.endswith((".cuh", ".h"))] + [os.path.join(ROOT, "include", "hprlp_b200.h")]
OUT = os.path.join(HERE, "libhprlp_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                 # every product/sum rounded separately, like numpy/scipy
    "-Xcompiler", "-fPIC", "-shared",
    "-diag-suppress", "177", "-Xcompiler", "-Wno-deprecated-declarations",
    "-ldl",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in DEPS)


HOST_SRC = os.path.join(HERE, "csrc", "hpr_host.cpp")


def host_out() -> str:
    import sysconfig
    return os.path.join(HERE, "_hpr_host" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def build_host(force: bool = False, verbose: bool = False) -> str | None:
    """The pybind11 host helpers (batch packing), g++ in-tree; None when the
    Python headers or pybind11 are unavailable (solve_batch then packs in numpy)."""
    import sysconfig
    try:
        import pybind11
    except ImportError:
        return None
    out = host_out()
    if not force and os.path.exists(out) and os.path.getmtime(out) > os.path.getmtime(HOST_SRC):
        return out
    cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++17", "-shared", "-fPIC", "-pthread",
           "-I" + sysconfig.get_paths()["include"], "-I" + pybind11.get_include(),
           "-o", out, HOST_SRC]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT, *SRC]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    build_host(force, verbose)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
