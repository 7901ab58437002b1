"""Build libhc.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import fcntl
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhc.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


# Diagnostic variant (timing experiments only, never loaded by default): -DHC_DIAG enables
# the wrong-output timing modes (HC_DIAG_EPI / HC_DIAG_BOX), -DHC_TIMELINE the fused kernel's
# per-CTA globaltimer stamps (hc_debug_timeline).  Loaded only with HC_LIB_VARIANT=diag.
VARIANTS = {"": ([], "libhc.so", "build"), "diag": (["-DHC_DIAG", "-DHC_TIMELINE"], "libhc_diag.so", "build_diag")}


def lib_path(variant: str = "") -> str:
    return os.path.join(HERE, VARIANTS[variant][1])


def needs_build(variant: str = "") -> bool:
    lib = lib_path(variant)
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps.append(os.path.join(os.path.dirname(HERE), "include", "hc.h"))
    return any(os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    """Compile if any source is newer than the library.  Concurrent callers (e.g. the ranks of
    a torchrun launch) serialise on a file lock: the first one builds, the others wait and
    then find the library up to date."""
    if not force and not needs_build(variant):
        return lib_path(variant)
    with open(os.path.join(HERE, ".build.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if not force and not needs_build(variant):
                return lib_path(variant)
            return _build_locked(verbose, variant)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


def _build_locked(verbose: bool, variant: str = "") -> str:
    defines, libname, objname = VARIANTS[variant]
    objdir = os.path.join(HERE, objname)
    os.makedirs(objdir, exist_ok=True)
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
                    "-I", os.path.join(os.path.dirname(HERE), "include")] + defines
    if verbose:
        flags += ["-Xptxas", "-v"]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen([nvcc()] + flags + ["-c", src, "-o", obj],
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    failed = False
    for p in procs:
        out, _ = p.communicate()
        if out and (verbose or p.returncode != 0):
            sys.stderr.write(out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    lib = os.path.join(HERE, libname)
    tmp = f"{lib}.{os.getpid()}.tmp"
    subprocess.check_call([nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart_static", "-ldl", "-lrt", "-lpthread"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant="diag" if "--diag" in sys.argv else ""))
