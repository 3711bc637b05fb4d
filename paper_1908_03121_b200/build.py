"""Build the sm_100a shared library libocto_fmm.so in-tree (nvcc, no JIT cache).

The library links the NCCL that ships with the torch wheel (nvidia/nccl), so
torch.distributed and the library use one NCCL in-process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libocto_fmm.so")
PEAK_LIB = os.path.join(HERE, "libocto_peak.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    cands = []
    for p in sys.path:
        cands += glob.glob(os.path.join(p, "nvidia", "nccl"))
    for c in cands:
        inc, lib = os.path.join(c, "include"), os.path.join(c, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted([f for f in glob.glob(os.path.join(CSRC, "*.cu")) if not f.endswith("fp64_peak.cu")] + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(CSRC, "*.hpp")) + [os.path.join(ROOT, "include", "octo_fmm.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build_peak(force: bool = False) -> str:
    """FP64 roofline probe (bench evidence), a separate tiny library."""
    src = os.path.join(CSRC, "fp64_peak.cu")
    if not force and os.path.exists(PEAK_LIB) and os.path.getmtime(PEAK_LIB) > os.path.getmtime(src):
        return PEAK_LIB
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC", src, "-o", PEAK_LIB]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-4000:])
    return PEAK_LIB


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra: list | None = None) -> str:
    """Build LIB (or, for tuning experiments, `out` with extra nvcc flags).

    Several processes (ranks of one job) may call this at once: the build is
    serialised by an exclusive lock on a file next to the library, and the
    staleness check is repeated under the lock, so one process builds and the
    others load its result."""
    if out is None and not force and not needs_build():
        return LIB
    import fcntl
    with open(os.path.join(HERE, ".build.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if out is None and not force and not needs_build():
            return LIB
        return _build_locked(verbose, out, extra)


def _build_locked(verbose: bool, out: str | None, extra: list | None) -> str:
    inc, lib = nccl_paths()
    libname = sorted(glob.glob(os.path.join(lib, "libnccl.so*")))[0]
    debug = ["-DOCTO_DEBUG"] if os.environ.get("OCTO_DEBUG_BUILD") == "1" else []
    # tuning builds only (e.g. "-DP2P_MINB=3"); the shipped library uses the defaults
    debug += os.environ.get("OCTO_NVCC_EXTRA", "").split() + list(extra or [])
    target = out or LIB
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", *debug,
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
           os.path.join(CSRC, "octo_fmm.cu"), os.path.join(CSRC, "exchange.cu"), os.path.join(CSRC, "upward.cu"),
           os.path.join(CSRC, "downward.cu"),
           "-o", target + f".tmp{os.getpid()}", "-Xlinker", libname, "-Xlinker", "-rpath=" + lib]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-6000:])
    os.replace(target + f".tmp{os.getpid()}", target)
    if verbose:
        print(res.stderr)
    return target


if __name__ == "__main__":
    build(force=True, verbose=True)
    build_peak(force=True)
