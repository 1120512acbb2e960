"""CPU: the C-ABI libraries load and export every declared entry point, the
Python mirror validates like the reference, and without a GPU the engine
refuses to run (there is no CPU fallback)."""
from __future__ import annotations

import ctypes
import re
import subprocess

import pytest

from conftest import HAS_GPU, ROOT

HEADER = ROOT / "include" / "bmmgpu.h"


def _declared() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(bmmgpu_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("bmmgpu_cubic", "bmmgpu_multiply", "bmmgpu_dev_cubic", "bmmgpu_dev_transpose",
                     "bmmgpu_basis_change", "bmmgpu_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    import paper_1909_01554_b200 as bmm
    lib = bmm.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(bmm.LIB_PATH)], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}$", out, re.M), name
    assert b"sm_100a" in lib.bmmgpu_version()


def test_python_mirror_declares_every_signature():
    """Every entry point with parameters has ctypes argtypes in the mirror (an undeclared
    one would pass 64-bit pointers and sizes as C ints)."""
    import paper_1909_01554_b200 as bmm
    lib = bmm.lib()
    text = HEADER.read_text()
    for name in _declared():
        params = re.search(rf"{name}\s*\(([^)]*)\)", text).group(1).strip()
        if params in ("", "void"):
            continue
        assert getattr(lib, name).argtypes is not None, name


def test_dropin_library_exports_the_bmm_api():
    import paper_1909_01554_b200 as bmm
    ctypes.CDLL(str(bmm.HOST_LIB_PATH))
    out = subprocess.run(["nm", "-DC", "--defined-only", str(bmm.HOST_LIB_PATH)], capture_output=True,
                         text=True).stdout
    for sym in ("bmm::multiply_cubic(", "bmm::multiply(", "bmm::multiply_alt(", "bmm::basis_change(",
                "bmm::BitMatrix::random(", "bmm::read_bmm1(", "bmm::write_bmm1(", "bmm::to_interleaved(",
                "bmm::from_interleaved(", "bmm::transpose_blocks64(", "bmm::kernel64(", "bmm::chain_multiply(",
                "bmm::LayerPlan::auto_plan(", "bmm::pad_pow2(", "bmm::interleaved_bit_index("):
        assert sym in out, sym


def test_kernels_are_sm100a_native():
    """The cubin carries tcgen05-era SASS for sm_100a only (no PTX JIT path)."""
    import paper_1909_01554_b200 as bmm
    out = subprocess.run(["cuobjdump", "--list-elf", str(bmm.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(bmm.LIB_PATH)], capture_output=True, text=True).stdout
    assert "LOP3.LUT" in sass
    # the default block product is a tcgen05 CTA-pair kernel fed by TMA: pair MMAs
    # (UTCOMMA.2CTA = tcgen05.mma.cta_group::2 kind::mxf4), TMEM loads / stores (LDTM /
    # STTM), the pair's TMEM allocator and commit barriers, 3-D tensor-map loads
    fns = sass.split("Function : ")
    k2 = [f for f in fns if "cubic_umma2_kernel" in f.splitlines()[0]]
    assert len(k2) == 4, "the TMA, TMA + A-in-TMEM, cp.async-loader and level-shifted (fold) instantiations"
    for op in ("UTCOMMA.2CTA", "LDTM", "STTM", "UTCATOMSWS.2CTA", "UTCBAR.2CTA"):
        assert all(op in f for f in k2), op
    assert sum("UTMALDG.3D" in f for f in k2) == 3  # TMA loaders: plain, A-in-TMEM and fold


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device path")
def test_no_cpu_fallback_without_device():
    import numpy as np
    import paper_1909_01554_b200 as bmm
    a = bmm.BitMatrix.zeros(64, 64)
    with pytest.raises(bmm.EngineError, match="no CUDA device"):
        bmm.multiply_cubic(a, a, bmm.Semiring.Gf2XorAnd)
    with pytest.raises(bmm.EngineError):
        bmm.multiply(a, a, bmm.Algo.AltSelfInverse, bmm.LayerPlan(), bmm.Semiring.Gf2XorAnd)
    assert np.array_equal(a.words, np.zeros(64, dtype=np.uint64))


def test_python_mirror_validates_like_the_reference():
    import paper_1909_01554_b200 as bmm
    a = bmm.BitMatrix.zeros(64, 65)
    b = bmm.BitMatrix.zeros(64, 64)
    with pytest.raises(bmm.ShapeError):
        bmm.multiply_cubic(a, b, bmm.Semiring.Gf2XorAnd)
    sq = bmm.BitMatrix.zeros(128, 128)
    with pytest.raises(ValueError):
        bmm.multiply(sq, sq, bmm.Algo.AltSelfInverse, bmm.LayerPlan.auto_plan(128, 1), bmm.Semiring.BooleanOrAnd)
    with pytest.raises(bmm.ShapeError):
        bmm.multiply(bmm.BitMatrix.zeros(96, 96), bmm.BitMatrix.zeros(96, 96), bmm.Algo.AltSelfInverse,
                     bmm.LayerPlan.auto_plan(128, 1), bmm.Semiring.Gf2XorAnd)
    with pytest.raises(ValueError):
        bmm.multiply(sq, sq, bmm.Algo.AltSelfInverse, bmm.LayerPlan.auto_plan(256, 1), bmm.Semiring.Gf2XorAnd)


def test_auto_plan_matches_reference():
    import paper_1909_01554_b200 as bmm
    # reference test_engine.cpp:199-224
    p = bmm.LayerPlan.auto_plan(64, 1)
    assert (p.d_host, p.d_serial, p.d_parallel, p.matrix_dim()) == (0, 0, 0, 64)
    p = bmm.LayerPlan.auto_plan(512, 4)
    assert (p.d_serial, p.d_parallel, p.workers) == (0, 3, 4)
    p = bmm.LayerPlan.auto_plan(4096, 2)
    assert (p.d_serial, p.d_parallel, p.matrix_dim()) == (3, 3, 4096)
    p = bmm.LayerPlan.auto_plan(16384, 0)
    assert (p.d_serial, p.d_parallel, p.workers) == (5, 3, 1)
    for bad in (96, 32, 0):
        with pytest.raises(bmm.ShapeError):
            bmm.LayerPlan.auto_plan(bad, 1)


def test_random_generator_matches_oracle(oracle):
    import numpy as np
    import paper_1909_01554_b200 as bmm
    for rows, cols, seed in [(130, 130, 7), (64, 64, 5), (3, 700, 9), (1000, 1, 4)]:
        m = bmm.BitMatrix.random(rows, cols, seed)
        assert np.array_equal(m.words, oracle.random(rows, cols, seed))


@pytest.mark.gpu
def test_init_warms_the_device_and_products_stay_exact(engine, oracle):
    """bmmgpu_init (every kernel once, stream pool, 1 GiB pool reserve) leaves the engine
    in a state where products are unchanged (alt-si through the level-shifted leaves)."""
    import numpy as np
    engine.init(0, 1 << 30)
    n = 1024
    a = oracle.random(n, n, 5)
    b = oracle.random(n, n, 6)
    got = engine.multiply(engine.BitMatrix(n, n, a), engine.BitMatrix(n, n, b), engine.Algo.AltSelfInverse,
                          engine.LayerPlan.auto_plan(n, 1), engine.Semiring.Gf2XorAnd, leaf_log2=8)
    assert np.array_equal(got.words, oracle.multiply_cubic(a, b, n, n, n, 1))
    with pytest.raises(ValueError):
        engine.init(1 << 30, 0)  # a device that does not exist
