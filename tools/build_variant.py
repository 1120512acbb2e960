#!/usr/bin/env python
"""Build an A/B variant of libbmmgpu.so with extra -D flags on one kernel source.

    python tools/build_variant.py NAME cubic_umma2.cu -DBMMGPU_GF2_PACK16=0 [...]

Writes build/variants/libbmmgpu_NAME.so (the other objects are the default build's
build/*.o, so run the default build first).  Experiment scripts under
tools/experiments/ swap it in for paper_1909_01554_b200/libbmmgpu.so on the GPU box.
"""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1909_01554_b200 import build as B  # noqa: E402


def main() -> None:
    name, src, *defs = sys.argv[1:]
    out = B.BUILD / "variants"
    out.mkdir(parents=True, exist_ok=True)
    obj = out / f"{Path(src).stem}_{name}.o"
    subprocess.run([B.NVCC, *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *defs,
                    "-I", str(ROOT / "include"), "-c", str(B.CSRC / src), "-o", str(obj)], check=True)
    objs = [obj if Path(s).stem == Path(src).stem else B.BUILD / (Path(s).stem + ".o") for s in B.CUDA_SOURCES]
    lib = out / f"libbmmgpu_{name}.so"
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
