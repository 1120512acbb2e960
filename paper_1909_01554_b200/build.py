"""Builds the in-tree native libraries for sm_100a.

    libbmmgpu.so   -- CUDA kernels + the extern "C" ABI (include/bmmgpu.h)
    libbmm_b200.so -- the C++ drop-in bmm:: API (include/bmm/*.hpp) over libbmmgpu.so

Both land next to this file so they travel with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
CSRC = HERE / "csrc"
BUILD = ROOT / "build"
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
CUDA_HOME = Path(NVCC).resolve().parent.parent
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CUDA_SOURCES = ["capi.cu", "transpose.cu", "cubic_lop3.cu", "cubic_umma2.cu", "alt.cu", "stream.cu", "bmm1.cu", "layout.cu", "alt_tiles.cu", "init.cu", "kernel64.cu"]
HOST_SOURCES = ["host/bitmatrix.cpp", "host/engine.cpp", "host/pipeline.cpp"]

LIB_GPU = HERE / "libbmmgpu.so"
LIB_HOST = HERE / "libbmm_b200.so"


def _run(cmd: list[str]) -> None:
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, jobs: int | None = None) -> None:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "bmmgpu.h"]
    objs = []
    procs = []
    for src in CUDA_SOURCES:
        s = CSRC / src
        o = BUILD / (Path(src).stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   "-I", str(ROOT / "include"), "-c", str(s), "-o", str(o)]
            print(" ".join(cmd), flush=True)
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        log = BUILD / (Path(src).stem + ".ptxas.log")
        log.write_text(out)
        if p.returncode != 0:
            print(out, file=sys.stderr)
            failed = True
    if failed:
        raise RuntimeError("nvcc failed")
    if force or _stale(LIB_GPU, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB_GPU), *map(str, objs), "-lcudart"])
    host_srcs = [CSRC / s for s in HOST_SOURCES]
    host_hdrs = list((ROOT / "include" / "bmm").glob("*.hpp")) + [ROOT / "include" / "bmmgpu.h"]
    if all(s.exists() for s in host_srcs) and (force or _stale(LIB_HOST, host_srcs + host_hdrs + [LIB_GPU])):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", str(ROOT / "include"),
              *map(str, host_srcs), "-o", str(LIB_HOST), "-L", str(HERE), "-lbmmgpu",
              f"-Wl,-rpath,$ORIGIN"])


if __name__ == "__main__":
    build(force="--force" in sys.argv)
