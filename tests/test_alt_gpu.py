"""GPU parity: the <2,2,2;7> fast products (Strassen-Winograd, alt-si,
alt-chain) on B200 equal the reference's outputs bit for bit, for every leaf
size the recursion can stop at."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

GF2 = 1
pytestmark = pytest.mark.gpu


def _plan(bmm, p):
    return bmm.LayerPlan(p[0], p[1], p[2], 1, 1)


@pytest.mark.parametrize("leaf", [0, 6, 7, 8, 10])
def test_fast_products_match_reference(engine, oracle, golden, leaf):
    bmm = engine
    for c in golden["fast"]:
        n = c["n"]
        if leaf and (64 << 0) * (1 << (leaf - 6)) > n:
            continue
        a = bmm.BitMatrix(n, n, oracle.random(n, n, c["a_seed"]))
        b = bmm.BitMatrix(n, n, oracle.random(n, n, c["b_seed"]))
        got = bmm.multiply(a, b, bmm.Algo(c["algo"]), _plan(bmm, c["plan"]), bmm.Semiring.Gf2XorAnd,
                           leaf_log2=leaf)
        assert f"{oracle.fnv1a64(got.words):016x}" == c["fnv"], (c, leaf)


def test_alt_equals_cubic_for_every_split(engine, oracle):
    bmm = engine
    for n in (64, 128, 256, 512):
        a = bmm.BitMatrix(n, n, oracle.random(n, n, 91 + n))
        b = bmm.BitMatrix(n, n, oracle.random(n, n, 92 + n))
        want = oracle.multiply_cubic(a.words, b.words, n, n, n, GF2)
        depth = (n // 64).bit_length() - 1
        for algo in (bmm.Algo.StrassenWinograd, bmm.Algo.AltSelfInverse, bmm.Algo.AltChaining):
            for ds in range(depth + 1):
                plan = bmm.LayerPlan(0, ds, depth - ds, 1, 1)
                got = bmm.multiply(a, b, algo, plan, bmm.Semiring.Gf2XorAnd, leaf_log2=6)
                assert np.array_equal(got.words, want), (n, algo, ds)


def test_single_bit_probes_cross_block_boundaries(engine):
    """reference test_engine.cpp:461-481."""
    bmm = engine
    plan = bmm.LayerPlan.auto_plan(128, 1)
    coords = (62, 63, 64, 65)
    for algo in (bmm.Algo.StrassenWinograd, bmm.Algo.AltSelfInverse, bmm.Algo.AltChaining):
        for i in coords:
            for j in coords:
                for k in coords:
                    eij, ejk, want = bmm.BitMatrix.zeros(128, 128), bmm.BitMatrix.zeros(128, 128), \
                        bmm.BitMatrix.zeros(128, 128)
                    eij.set(i, j, True)
                    ejk.set(j, k, True)
                    want.set(i, k, True)
                    assert bmm.multiply(eij, ejk, algo, plan, bmm.Semiring.Gf2XorAnd, leaf_log2=6) == want


def test_identity_and_associativity(engine, oracle):
    bmm = engine
    plan = bmm.LayerPlan.auto_plan(256, 1)
    c, d, e = (bmm.BitMatrix(256, 256, oracle.random(256, 256, s)) for s in (95, 96, 97))
    alt = bmm.Algo.AltSelfInverse
    cd = bmm.multiply(c, d, alt, plan, bmm.Semiring.Gf2XorAnd, leaf_log2=6)
    de = bmm.multiply(d, e, alt, plan, bmm.Semiring.Gf2XorAnd, leaf_log2=6)
    assert bmm.multiply(cd, e, alt, plan, bmm.Semiring.Gf2XorAnd, leaf_log2=7) == \
        bmm.multiply(c, de, alt, plan, bmm.Semiring.Gf2XorAnd, leaf_log2=7)
    ident = bmm.BitMatrix.zeros(256, 256)
    for i in range(256):
        ident.set(i, i, True)
    for algo in (bmm.Algo.StrassenWinograd, bmm.Algo.AltSelfInverse, bmm.Algo.AltChaining):
        assert bmm.multiply(c, ident, algo, plan, bmm.Semiring.Gf2XorAnd, leaf_log2=6) == c
        assert bmm.multiply(ident, c, algo, plan, bmm.Semiring.Gf2XorAnd, leaf_log2=6) == c


def test_large_alt_si_against_golden(engine, oracle, golden):
    """n=4096 alt-si (reference plan 3 serial + 3 parallel) == the cubic digest."""
    bmm = engine
    c = next(x for x in golden["fast"] if x["n"] == 4096)
    cub = next(x for x in golden["cubic_large"] if x["m"] == 4096 and x["ring"] == GF2)
    assert c["fnv"] == cub["fnv"]
    a = bmm.BitMatrix(4096, 4096, oracle.random(4096, 4096, 1))
    b = bmm.BitMatrix(4096, 4096, oracle.random(4096, 4096, 2))
    for leaf in (0, 9, 10, 11):
        got = bmm.multiply(a, b, bmm.Algo.AltSelfInverse, _plan(bmm, c["plan"]), bmm.Semiring.Gf2XorAnd,
                           leaf_log2=leaf)
        assert f"{oracle.fnv1a64(got.words):016x}" == c["fnv"], leaf


def test_interleaved_basis_change_matches_reference(engine, oracle, golden):
    bmm = engine
    lib = bmm.lib()
    v = oracle.random(1, 4 * 4 * 4096, 41)
    algo_of_scheme = {1: 2, 2: 3}  # bmm::Builtin -> bmm::Algo id
    for c in golden["basis_change"]:
        w = v.copy()
        assert lib.bmmgpu_basis_change(w.ctypes.data, w.size, 2, algo_of_scheme[c["scheme"]], c["which"], 0) == 0
        assert f"{oracle.fnv1a64(w):016x}" == c["fnv"], c
        assert lib.bmmgpu_basis_change(w.ctypes.data, w.size, 2, algo_of_scheme[c["scheme"]], c["which"], 1) == 0
        assert np.array_equal(w, v)


@pytest.mark.parametrize("serial", [1, 2, 3])
def test_depth_first_levels_match_reference(engine, oracle, golden, serial, monkeypatch):
    """The top `serial` recursion levels run depth-first (children formed, multiplied
    and folded one at a time), the rest breadth-first: same bits for every split."""
    bmm = engine
    monkeypatch.setenv("BMMGPU_ALT_SERIAL", str(serial))
    for c in golden["fast"]:
        n = c["n"]
        a = bmm.BitMatrix(n, n, oracle.random(n, n, c["a_seed"]))
        b = bmm.BitMatrix(n, n, oracle.random(n, n, c["b_seed"]))
        for leaf in (6, 7):
            got = bmm.multiply(a, b, bmm.Algo(c["algo"]), _plan(bmm, c["plan"]), bmm.Semiring.Gf2XorAnd,
                               leaf_log2=leaf)
            assert f"{oracle.fnv1a64(got.words):016x}" == c["fnv"], (c, leaf, serial)


@pytest.mark.parametrize("leaf", [6, 7, 8])
def test_device_fast_product_reads_operands_only(engine, oracle, leaf):
    """bmmgpu_dev_multiply on torch-owned HBM: equal to the cubic product for every
    scheme, and dA / dBt come back unchanged (the basis changes are folded into the
    expand / compress coefficients, not applied in place)."""
    import ctypes

    import torch
    bmm = engine
    lib = bmm.lib()
    n = 1024
    a = oracle.random(n, n, 71)
    b = oracle.random(n, n, 72)
    want = oracle.multiply_cubic(a, b, n, n, n, GF2)
    w = n // 64
    dA = torch.from_numpy(a.view(np.int64).reshape(n, w).copy()).cuda()
    dB = torch.from_numpy(b.view(np.int64).reshape(n, w).copy()).cuda()
    dBt = torch.empty((n, w), dtype=torch.int64, device="cuda")
    dC = torch.empty((n, w), dtype=torch.int64, device="cuda")
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.bmmgpu_dev_transpose(dB.data_ptr(), w, n, n, dBt.data_ptr(), n, w, stream) == 0
    bt0 = dBt.clone()
    for algo in (1, 2, 3):
        assert lib.bmmgpu_dev_multiply(dA.data_ptr(), w, dBt.data_ptr(), w, dC.data_ptr(), w, n, algo, leaf, 0,
                                       stream) == 0
        torch.cuda.synchronize()
        assert np.array_equal(dC.cpu().numpy().view(np.uint64).ravel(), want), (algo, leaf)
        assert np.array_equal(dA.cpu().numpy().view(np.uint64).ravel(), a)
        assert torch.equal(dBt, bt0)


@pytest.mark.parametrize("n,leaf,levels", [(1024, 6, None), (1024, 8, None), (1024, 6, "2"), (1024, 8, "2"),
                                           (2048, 8, "2"), (2048, 7, "2"), (2048, 8, "1"), (2048, 7, "1"),
                                           (2048, 7, "3"), (1024, 6, "3")])
def test_streamed_host_path_pinned_buffers(engine, oracle, monkeypatch, n, leaf, levels):
    """bmmgpu_multiply from page-locked host buffers: the streamed driver uploads A / B
    quadrant by quadrant (e = 2, or BMMGPU_ALT_STREAM_LEVELS=1) or sub-block by sub-block
    (e >= 3: every child as its 7 grandchildren at n >= 2^17 or with =2, the first and
    last child only below that or with =3) behind the first products and downloads each part of
    C as soon as it is final; same bits as the cubic product for every scheme."""
    import torch
    bmm = engine
    if levels:
        monkeypatch.setenv("BMMGPU_ALT_STREAM_LEVELS", levels)
    a = oracle.random(n, n, 81)
    b = oracle.random(n, n, 82)
    want = oracle.multiply_cubic(a, b, n, n, n, GF2)
    ha = torch.from_numpy(a.view(np.int64)).pin_memory()
    hb = torch.from_numpy(b.view(np.int64)).pin_memory()
    hc = torch.zeros(n * n // 64, dtype=torch.int64).pin_memory()
    for algo in (bmm.Algo.StrassenWinograd, bmm.Algo.AltSelfInverse, bmm.Algo.AltChaining):
        out = bmm.BitMatrix(n, n, hc.numpy().view(np.uint64))
        got = bmm.multiply(bmm.BitMatrix(n, n, ha.numpy().view(np.uint64)),
                           bmm.BitMatrix(n, n, hb.numpy().view(np.uint64)), algo, bmm.LayerPlan.auto_plan(n, 1),
                           bmm.Semiring.Gf2XorAnd, leaf_log2=leaf, out=out)
        assert np.array_equal(got.words, want), (algo, leaf)


@pytest.mark.parametrize("budget", [None, 64 << 10, 16 << 10, 4 << 10])
def test_interleaved_basis_change_streams_beyond_the_budget(engine, oracle, monkeypatch, budget):
    """bmmgpu_basis_change on vectors larger than the device budget (the standalone
    transform at 2^20 is 128 GiB): levels whose groups exceed a device block stream as
    strided passes, the rest in one blocked pass -- same words as the in-core run, and
    the inverse restores the input."""
    lib = engine.lib()
    levels = 4
    v = oracle.random(1, (4 ** levels) * 4096, 43)  # [4]^4 [4096]: 128 KiB
    want = {}
    for algo, factor in ((2, 0), (2, 2), (3, 0), (3, 1), (3, 2)):
        w = v.copy()
        monkeypatch.delenv("BMMGPU_BASIS_BUDGET", raising=False)
        assert lib.bmmgpu_basis_change(w.ctypes.data, w.size, levels, algo, factor, 0) == 0
        want[(algo, factor)] = w
    if budget is not None:
        monkeypatch.setenv("BMMGPU_BASIS_BUDGET", str(budget))
    for (algo, factor), ref in want.items():
        w = v.copy()
        assert lib.bmmgpu_basis_change(w.ctypes.data, w.size, levels, algo, factor, 0) == 0
        assert np.array_equal(w, ref), (algo, factor, budget)
        assert lib.bmmgpu_basis_change(w.ctypes.data, w.size, levels, algo, factor, 1) == 0
        assert np.array_equal(w, v), (algo, factor, budget)


@pytest.mark.parametrize("budget", [None, 24 << 10, 6 << 10])
def test_basis_change_inner_mode_not_power_of_two(engine, oracle, monkeypatch, budget):
    """[4]*3 [7 * 4096 bits] vectors (the inner mode is not a power of two; reference
    basis_change accepts them, engine.cpp:146-172): streamed blocks are whole level
    groups, so the result equals the in-core run and the inverse restores the input."""
    lib = engine.lib()
    levels, inner = 3, 7 * 64
    v = oracle.random(1, (4 ** levels) * inner * 64, 47)
    monkeypatch.delenv("BMMGPU_BASIS_BUDGET", raising=False)
    want = v.copy()
    assert lib.bmmgpu_basis_change(want.ctypes.data, want.size, levels, 2, 0, 0) == 0
    # phi of alt-si applied level by level in numpy: x11 ^= x01 ^ x10 over [outer][4][inner_l]
    ref = v.copy()
    for l in range(levels):
        il = v.size >> (2 * (l + 1))
        r = ref.reshape(-1, 4, il)
        r[:, 3] ^= r[:, 1] ^ r[:, 2]
    assert np.array_equal(want, ref)
    if budget is not None:
        monkeypatch.setenv("BMMGPU_BASIS_BUDGET", str(budget))
    w = v.copy()
    assert lib.bmmgpu_basis_change(w.ctypes.data, w.size, levels, 2, 0, 0) == 0
    assert np.array_equal(w, want), budget
    assert lib.bmmgpu_basis_change(w.ctypes.data, w.size, levels, 2, 0, 1) == 0
    assert np.array_equal(w, v), budget


def test_multiply_alt_hat_vectors_match_reference_digests(engine, oracle, golden):
    """bmmgpu_multiply_alt (the reference's multiply_alt on interleaved vectors already in
    the scheme's basis, engine.cpp:293-349, and the solve stage of the host pipeline)
    reproduces the reference's own outputs: FNV digests, popcounts and first words from
    oracle/_ref for all three schemes, depths 2 to 5."""
    lib = engine.lib()
    for c in golden["multiply_alt"]:
        depth = c["d_serial"] + c["d_parallel"]
        n = 64 << depth
        ah = oracle.random(1, n * n, c["a_seed"])
        bh = oracle.random(1, n * n, c["b_seed"])
        ch = np.zeros_like(ah)
        for leaf in (0, 7):  # default leaves, and 128-bit leaves (more recursion levels on the GPU)
            opts = engine._opts(0, leaf_log2=leaf)
            assert lib.bmmgpu_multiply_alt(ah.ctypes.data, bh.ctypes.data, ch.ctypes.data, depth, c["scheme"] + 1,
                                           ctypes.byref(opts)) == 0, lib.bmmgpu_last_error()
            assert f"{oracle.fnv1a64(ch):016x}" == c["fnv"], (c, leaf)
            assert oracle.popcount(ch) == c["pop"] and f"{int(ch[0]):016x}" == c["w0"]


@pytest.mark.parametrize("driver", ["subinst", "tiles"])
@pytest.mark.parametrize("n,tile,leaf", [(1024, 8, 6), (2048, 9, 7), (2048, 10, 8), (4096, 11, 9), (1024, 10, 7), (1024, 9, 12)])
def test_out_of_core_tiles_equal_cubic(engine, oracle, monkeypatch, n, tile, leaf, driver):
    """The out-of-core fast products, forced at small n, from pageable and page-locked
    buffers, for every scheme: the bits of the cubic product.  subinst (the one-device
    default, alt.cu): the recursion's top-level sub-instances generated on the device from
    streamed source sub-blocks, Q folded into C by host threads; tiles (alt_tiles.cu): C
    tiles = XOR over K of alt-basis block products of streamed tiles."""
    import torch
    bmm = engine
    monkeypatch.setenv("BMMGPU_ALT_TILE", str(tile))
    if driver == "tiles":
        monkeypatch.setenv("BMMGPU_ALT_OOC", "tiles")
    else:
        monkeypatch.delenv("BMMGPU_ALT_OOC", raising=False)
    a = oracle.random(n, n, 91)
    b = oracle.random(n, n, 92)
    want = oracle.multiply_cubic(a, b, n, n, n, GF2)
    for algo in (bmm.Algo.StrassenWinograd, bmm.Algo.AltSelfInverse, bmm.Algo.AltChaining):
        got = bmm.multiply(bmm.BitMatrix(n, n, a), bmm.BitMatrix(n, n, b), algo, bmm.LayerPlan.auto_plan(n, 1),
                           bmm.Semiring.Gf2XorAnd, leaf_log2=leaf, force_streaming=True)
        assert np.array_equal(got.words, want), (algo, n, tile)
    ha = torch.from_numpy(a.view(np.int64)).pin_memory()
    hb = torch.from_numpy(b.view(np.int64)).pin_memory()
    hc = torch.zeros(n * n // 64, dtype=torch.int64).pin_memory()
    got = bmm.multiply(bmm.BitMatrix(n, n, ha.numpy().view(np.uint64)), bmm.BitMatrix(n, n, hb.numpy().view(np.uint64)),
                       bmm.Algo.AltSelfInverse, bmm.LayerPlan.auto_plan(n, 1), bmm.Semiring.Gf2XorAnd,
                       leaf_log2=leaf, force_streaming=True, out=bmm.BitMatrix(n, n, hc.numpy().view(np.uint64)))
    assert np.array_equal(got.words, want)


@pytest.mark.parametrize("driver", ["subinst", "tiles"])
def test_out_of_core_tiles_by_budget(engine, oracle, monkeypatch, driver):
    """A device budget below six n^2/8 arrays selects the out-of-core driver without the
    force flag (golden n = 4096 alt-si product of the reference's seeds)."""
    bmm = engine
    monkeypatch.setenv("BMMGPU_ALT_TILE", "11")
    if driver == "tiles":
        monkeypatch.setenv("BMMGPU_ALT_OOC", "tiles")
    else:
        monkeypatch.delenv("BMMGPU_ALT_OOC", raising=False)
    n = 4096
    a = oracle.random(n, n, 1)
    b = oracle.random(n, n, 2)
    want = oracle.multiply_cubic(a, b, n, n, n, GF2)
    got = bmm.multiply(bmm.BitMatrix(n, n, a), bmm.BitMatrix(n, n, b), bmm.Algo.AltSelfInverse,
                       bmm.LayerPlan.auto_plan(n, 1), bmm.Semiring.Gf2XorAnd, leaf_log2=9,
                       device_budget=6 * n * n // 8 - 1)
    assert np.array_equal(got.words, want)
    assert engine.lib().bmmgpu_last_launch_count() > 8  # 2 x 2 tiles x 2 K-blocks


@pytest.mark.parametrize("leaf", [8, 9, 10, 12])
def test_level_shifted_leaves_match_reference(engine, oracle, golden, monkeypatch, leaf):
    """K2 fold mode (BMMGPU_ALT_FOLD=1: the last expand level formed inside the leaf
    kernel from the parents' quadrants, reference fused_block_stage engine.cpp:202-228)
    gives the reference's bits for every scheme; at leaf 12 with n = 4096 the parents are
    the operands themselves (e = 1)."""
    monkeypatch.setenv("BMMGPU_ALT_FOLD", "1")
    test_fast_products_match_reference(engine, oracle, golden, leaf)
    bmm = engine
    for n, seed in ((4096, 1), (2048, 7)):
        a = oracle.random(n, n, seed)
        b = oracle.random(n, n, seed + 1)
        want = oracle.multiply_cubic(a, b, n, n, n, GF2)
        for algo in (bmm.Algo.StrassenWinograd, bmm.Algo.AltSelfInverse, bmm.Algo.AltChaining):
            got = bmm.multiply(bmm.BitMatrix(n, n, a), bmm.BitMatrix(n, n, b), algo, bmm.LayerPlan.auto_plan(n, 1),
                               bmm.Semiring.Gf2XorAnd, leaf_log2=leaf)
            assert np.array_equal(got.words, want), (algo, n, leaf)


@pytest.mark.parametrize("algo", [1, 2, 3])
def test_production_leaves_every_scheme_against_reference_digest(engine, oracle, golden, algo):
    """The production leaf size (4096-bit leaves on the tcgen05 kernel) for sw, alt-si and
    alt-chain: n = 8192 (one recursion level) must reproduce the reference's own n = 8192
    GF(2) product digest (golden cubic_large, seeds 1 and 2); n = 16384 (one fused
    two-level expand / compress pass around 49 leaves) must equal the cubic product of the
    same operands and pass Freivalds-style row checks in numpy."""
    bmm = engine
    cub = next(x for x in golden["cubic_large"] if x["m"] == 8192 and x["ring"] == GF2)
    a = bmm.BitMatrix(8192, 8192, oracle.random(8192, 8192, cub["a_seed"]))
    b = bmm.BitMatrix(8192, 8192, oracle.random(8192, 8192, cub["b_seed"]))
    plan = bmm.LayerPlan.auto_plan(8192, 1)
    got = bmm.multiply(a, b, bmm.Algo(algo), plan, bmm.Semiring.Gf2XorAnd, leaf_log2=12)
    assert f"{oracle.fnv1a64(got.words):016x}" == cub["fnv"], algo
    n = 16384
    a = bmm.BitMatrix(n, n, oracle.random(n, n, 41))
    b = bmm.BitMatrix(n, n, oracle.random(n, n, 42))
    got = bmm.multiply(a, b, bmm.Algo(algo), bmm.LayerPlan.auto_plan(n, 1), bmm.Semiring.Gf2XorAnd, leaf_log2=12)
    want = bmm.multiply_cubic(a, b, bmm.Semiring.Gf2XorAnd)
    assert np.array_equal(got.words, want.words), algo
    B = b.words.reshape(n, n // 64)
    for i in (0, 4097, n - 1):
        bits = np.unpackbits(a.words.reshape(n, n // 64)[i].view(np.uint8), bitorder="little")
        assert np.array_equal(got.words.reshape(n, n // 64)[i], np.bitwise_xor.reduce(B[np.flatnonzero(bits)], axis=0))



@pytest.mark.parametrize("d_host", [1, 2, 3])
def test_out_of_core_subinstances_with_host_levels(engine, oracle, d_host):
    """The sub-instance driver with the caller's host levels (plan.d_host = 1..3: 7, 49, 343
    sub-instances, several selecting up to 4^d_host source sub-blocks each), every scheme,
    page-locked buffers: the bits of the cubic product."""
    import torch
    bmm = engine
    n = 4096
    depth = (n // 64).bit_length() - 1
    a = oracle.random(n, n, 97)
    b = oracle.random(n, n, 98)
    want = oracle.multiply_cubic(a, b, n, n, n, GF2)
    ha = torch.from_numpy(a.view(np.int64)).pin_memory()
    hb = torch.from_numpy(b.view(np.int64)).pin_memory()
    for algo in (1, 2, 3):
        hc = torch.zeros(n * n // 64, dtype=torch.int64).pin_memory()
        plan = bmm._Plan(d_host, depth - d_host, 0, 1, 1)
        opts = bmm._opts(0, leaf_log2=8, force_streaming=True)
        assert bmm.lib().bmmgpu_multiply(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), n, algo, ctypes.byref(plan), GF2,
                                         ctypes.byref(opts)) == 0, bmm.lib().bmmgpu_last_error()
        assert np.array_equal(hc.numpy().view(np.uint64), want), (algo, d_host)


def test_out_of_core_subinstances_staged_pieces_match_in_core(engine, oracle):
    """n = 32768 out of core through the sub-instance driver from pageable buffers, where every
    piece (16384 x 16384 bits, 32 MiB) goes through the page-locked staging slots: equal to the
    in-core fast product of the same operands and to numpy rows of A.B."""
    bmm = engine
    n = 32768
    a = oracle.random(n, n, 121)
    b = oracle.random(n, n, 122)
    plan = bmm.LayerPlan.auto_plan(n, 1)
    want = bmm.multiply(bmm.BitMatrix(n, n, a), bmm.BitMatrix(n, n, b), bmm.Algo.AltSelfInverse, plan,
                        bmm.Semiring.Gf2XorAnd)
    got = bmm.multiply(bmm.BitMatrix(n, n, a), bmm.BitMatrix(n, n, b), bmm.Algo.AltSelfInverse, plan,
                       bmm.Semiring.Gf2XorAnd, force_streaming=True)
    assert np.array_equal(got.words, want.words)
    B = b.reshape(n, n // 64)
    for i in (0, 12345, n - 1):
        bits = np.unpackbits(a.reshape(n, n // 64)[i].view(np.uint8), bitorder="little")
        assert np.array_equal(got.words.reshape(n, n // 64)[i], np.bitwise_xor.reduce(B[np.flatnonzero(bits)], axis=0))


@pytest.mark.parametrize("leaf", [7, 8, 9, 10])
@pytest.mark.parametrize("setting", [
    {"BMMGPU_ALT_NO_STREAM": "1", "BMMGPU_ALT_OVERLAP": "0"},
    {"BMMGPU_ALT_NO_STREAM": "1", "BMMGPU_ALT_OVERLAP": "1"},
    {"BMMGPU_ALT_NO_STREAM": "1", "BMMGPU_ALT_OVERLAP": "1", "BMMGPU_ALT_OVERLAP_ORDER": "1"},
    {"BMMGPU_ALT_NO_STREAM": "1", "BMMGPU_ALT_OVERLAP": "3", "BMMGPU_ALT_OVERLAP_MIN": "1"},
    {"BMMGPU_ALT_OVERLAP": "1", "BMMGPU_ALT_OVERLAP_MIN": "1"},  # streamed host path, grouped children
])
def test_overlapped_leaf_groups_match_reference(engine, oracle, golden, monkeypatch, leaf, setting):
    """The overlapped leaf groups (alt.cu alt_breadth: the last expand / first compress pass
    per group of leaves on a second stream beside the leaf launches, some CTA pairs left
    idle) against the plain breadth-first order: n = 8192 with leaves 2^7..2^10 (e = 6, 5,
    4, 3 levels: two-level and single-level passes above the groups, padded leaf panels at
    2^7) must reproduce the reference's own n = 8192 GF(2) digest for every scheme, in both
    pass orders, with groups as small as 49 leaves, in core and inside the streamed host
    path's children."""
    for k, v in setting.items():
        monkeypatch.setenv(k, v)
    bmm = engine
    cub = next(x for x in golden["cubic_large"] if x["m"] == 8192 and x["ring"] == GF2)
    a = bmm.BitMatrix(8192, 8192, oracle.random(8192, 8192, cub["a_seed"]))
    b = bmm.BitMatrix(8192, 8192, oracle.random(8192, 8192, cub["b_seed"]))
    for algo in (bmm.Algo.StrassenWinograd, bmm.Algo.AltSelfInverse, bmm.Algo.AltChaining):
        got = bmm.multiply(a, b, algo, bmm.LayerPlan.auto_plan(8192, 1), bmm.Semiring.Gf2XorAnd, leaf_log2=leaf)
        assert f"{oracle.fnv1a64(got.words):016x}" == cub["fnv"], (algo, leaf, setting)
