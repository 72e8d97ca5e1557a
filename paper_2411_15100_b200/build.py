"""Build libgmask.so in-tree with nvcc for sm_100a.

The library is a plain C-ABI shared object (include/gmask.h); it is loaded
with ctypes, so it carries no torch types.  The built .so lives next to this
file and travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libgmask.so"
BUILD = PKG / "_build"

SOURCES = ["gm_api.cu", "k_apply.cu", "k_cache.cu", "k_fill.cu", "k_accept.cu"]
HOST_SOURCES = ["front_end.cpp", "grammar_parse.cpp"]  # host-only C++ (g++)
HEADERS = ["common.cuh", "device.cuh", "accept.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libgmask.so")
    return cand


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HOST_SOURCES + HEADERS] + [ROOT / "include" / "gmask.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: Path = None) -> Path:
    global OUT
    if out is not None:  # diagnostics: variant builds into another file
        OUT, saved = Path(out), OUT
        try:
            return build(force=True, verbose=verbose)
        finally:
            OUT = saved
    if not force and not _stale():
        return OUT
    # several processes (torchrun ranks) may find the library stale at once:
    # one builds, the others wait on the lock and then see it fresh
    import fcntl

    BUILD.mkdir(exist_ok=True)
    with open(BUILD / ".build.lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and not _stale():
            return OUT
        return _build_locked(verbose)


def _build_locked(verbose: bool) -> Path:
    nvcc = _nvcc()
    BUILD.mkdir(exist_ok=True)
    include = ["-I", str(ROOT / "include"), "-I", str(CSRC)]
    if os.environ.get("GMASK_TIMELINE") == "1":  # diagnostics build: per-CTA timeline + CTA-0 phase marks
        include += ["-DGM_TIMELINE", "-DGM_TRACE_MARKS"]
    if os.environ.get("GMASK_PROBES") == "1":  # debug: K5 dry-walk / load-latency probes (GMASK_TRACE=1)
        include += ["-DGM_TRACE_PROBES"]
    if os.environ.get("GMASK_VERIFY") == "1":  # debug: cross-check cached arena keys
        include += ["-DGM_VERIFY_KNOWN"]

    extra = os.environ.get("GMASK_NVCC_EXTRA", "").split()  # diagnostics: variant builds

    def compile_one(src: str):
        obj = BUILD / (Path(src).stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra, *include, "-c", str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        (BUILD / (Path(src).stem + ".ptxas.txt")).write_text(res.stderr)
        return obj

    def compile_host(src: str):
        obj = BUILD / (Path(src).stem + ".o")
        cxx = shutil.which("g++") or "g++"
        cmd = [cxx, "-O2", "-std=c++17", "-fPIC", "-Wall", *include, "-c", str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"g++ failed for {src}:\n{res.stderr}")
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES) + len(HOST_SOURCES)) as ex:
        futs = [ex.submit(compile_one, s) for s in SOURCES] + [ex.submit(compile_host, s) for s in HOST_SOURCES]
        objs = [f.result() for f in futs]
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *map(str, objs), "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, OUT)
    if verbose:
        for src in SOURCES:
            print((BUILD / (Path(src).stem + ".ptxas.txt")).read_text(), file=sys.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
