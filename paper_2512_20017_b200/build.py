"""In-tree build of the sm_100a kernel library (and the CPU oracle used by the
tests).  Plain nvcc/gcc invocations; outputs are git-ignored .so files that
travel to the GPU box with the gpurun snapshot."""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libsplat_b200.so")
HOST_LIB = os.path.join(LIBDIR, "libsplat_host.so")
HOST_SOURCES = ["host/partition.cpp", "host/placement.cpp"]
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_LIB = os.path.join(ORACLE_DIR, "build", "libsplat_oracle.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr",
]
SOURCES = ["abi.cu", "cull.cu", "sort.cu", "project.cu", "bin.cu", "bin_tiles.cu", "raster.cu", "raster2d.cu", "patches.cu", "peer.cu", "densify.cu", "views.cu"]
HEADERS = ["common.cuh", "splat_math.cuh", "splat2d_math.cuh", "tile.cuh", "packed.cuh"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (res.stdout or res.stderr):
        sys.stderr.write(res.stdout + res.stderr)


def build_native(force: bool = False, verbose: bool = False, extra_flags=()) -> str:
    """Compile csrc/*.cu for sm_100a and link libsplat_b200.so (in-tree)."""
    os.makedirs(os.path.join(LIBDIR, "obj"), exist_ok=True)
    header = os.path.join(ROOT, "include", "splat_b200.h")
    common = [os.path.join(CSRC, h) for h in HEADERS] + [header]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(LIBDIR, "obj", src.replace(".cu", ".o"))
        objs.append(o)
        if force or not _newer(o, [s] + common):
            jobs.append([NVCC, *NVCC_FLAGS, *extra_flags, "-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    if force or jobs or not _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"], verbose)
    return LIB


def build_host(force: bool = False, verbose: bool = False) -> str:
    """Compile the host-side scheduling library (C++, no CUDA) in-tree."""
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in HOST_SOURCES]
    hdr = os.path.join(ROOT, "include", "splat_host.h")
    if force or not _newer(HOST_LIB, srcs + [hdr]):
        _run(["g++", "-O3", "-std=c++17", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-Wall", "-o", HOST_LIB,
              *srcs], verbose)
    return HOST_LIB


def build_oracle(force: bool = False, verbose: bool = False) -> str:
    """Compile the CPU oracle (test infrastructure only) with gcc."""
    src = os.path.join(ORACLE_DIR, "splat_oracle.c")
    hdr = os.path.join(ORACLE_DIR, "splat_oracle.h")
    os.makedirs(os.path.dirname(ORACLE_LIB), exist_ok=True)
    if force or not _newer(ORACLE_LIB, [src, hdr]):
        _run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
              "-fPIC", "-shared", "-o", ORACLE_LIB, src, "-lm"], verbose)
    return ORACLE_LIB


if __name__ == "__main__":
    v = "-v" in sys.argv
    f = "-f" in sys.argv
    # BS_NVCC_EXTRA: extra nvcc flags for tuning experiments (e.g. -DBS_SPARSE_LANES=5)
    print(build_native(force=f, verbose=v, extra_flags=os.environ.get("BS_NVCC_EXTRA", "").split()))
    print(build_host(force=f, verbose=v))
    if os.path.exists(os.path.join(ORACLE_DIR, "splat_oracle.c")):
        print(build_oracle(force=f, verbose=v))
