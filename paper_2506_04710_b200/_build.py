"""Builds libtbt.so (sm_100a CUDA + C++ host, the product) in-tree.

nvcc compiles each translation unit for `-gencode arch=compute_100a,
code=sm_100a` with -lineinfo (so ncu's source page maps to the code) and
links one shared library with a static cudart. No torch extension: the
boundary is the C ABI of include/tbt.h.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
BUILD = REPO / "build" / "tbt"
LIB = PKG / "libtbt.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-Wall",
    "--expt-relaxed-constexpr", "-Xptxas", "-v",
    f"-I{REPO / 'include'}", f"-I{CSRC}",
]
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", "-Wextra", f"-I{REPO / 'include'}"]


def _sources():
    return sorted(CSRC.glob("*.cu")), sorted(CSRC.glob("*.cpp"))


def _needs(obj: Path, deps) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    cus, cpps = _sources()
    headers = list(CSRC.glob("*.cuh")) + list((REPO / "include").glob("*.h"))
    jobs = []
    for src in cus:
        obj = BUILD / (src.stem + ".o")
        if force or _needs(obj, [src, *headers]):
            jobs.append([NVCC, *NVFLAGS, "-c", str(src), "-o", str(obj)])
    for src in cpps:
        obj = BUILD / (src.stem + ".cpp.o")
        if force or _needs(obj, [src, *headers]):
            jobs.append(["g++", *CXXFLAGS, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for cmd, r in ex.map(run, jobs):
            log = BUILD / (Path(cmd[-1]).name + ".log")
            log.write_text(r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"compile failed: {' '.join(cmd)}")
            if verbose:
                sys.stderr.write(r.stderr)
    objs = [BUILD / (s.stem + ".o") for s in cus] + [BUILD / (s.stem + ".cpp.o") for s in cpps]
    if force or _needs(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


def build_oracle() -> None:
    """Test infrastructure: CPU oracle + oracle/_ref (reference fft.cpp)."""
    r = subprocess.run(["make", "-C", str(REPO / "oracle")], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("oracle build failed")


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    build_oracle()
    print(LIB)
