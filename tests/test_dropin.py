"""The C++ drop-in (include/bmm/*.hpp + libbmm_b200.so): a C++ program written
against the reference's header API, compiled here with g++ and run -- host
cases on CPU, product cases on the GPU (-m gpu)."""
from __future__ import annotations

import subprocess

import pytest

from conftest import HAS_GPU, ROOT

SRC = ROOT / "tests" / "cpp" / "test_dropin.cpp"
BIN = ROOT / "build" / "test_dropin"


@pytest.fixture(scope="module")
def dropin_binary():
    import paper_1909_01554_b200 as bmm
    lib_dir = bmm.HOST_LIB_PATH.parent
    if not BIN.exists() or BIN.stat().st_mtime < max(SRC.stat().st_mtime, bmm.HOST_LIB_PATH.stat().st_mtime):
        BIN.parent.mkdir(exist_ok=True)
        subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), str(SRC), "-o", str(BIN),
                        "-L", str(lib_dir), "-lbmm_b200", "-lbmmgpu", f"-Wl,-rpath,{lib_dir}"], check=True)
    return BIN


def _run(binary, mode: str, env: dict | None = None) -> str:
    import os
    r = subprocess.run([str(binary), mode], capture_output=True, text=True, cwd=str(ROOT / "build"), timeout=600,
                       env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


def test_dropin_host_api(dropin_binary):
    out = _run(dropin_binary, "host")
    assert "0 failures" in out


@pytest.mark.gpu
@pytest.mark.skipif(not HAS_GPU, reason="no CUDA device")
@pytest.mark.parametrize("pipeline", ["device", "host"])
def test_dropin_products_on_gpu(dropin_binary, pipeline):
    """The reference suites' product cases through the drop-in; `pipeline::coordinate`
    runs its host layer on the device when the operands fit (default) and as the
    host-thread pipeline with BMM_PIPELINE=host -- both against the reference's outputs
    and counters."""
    out = _run(dropin_binary, "gpu", {"BMM_PIPELINE": pipeline})
    for line in out.splitlines():
        if line.startswith("C6:"):  # the reference's soft crossover criterion, reported not asserted
            print(line)
    assert "0 failures" in out
