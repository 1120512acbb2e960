"""GPU parity: the cubic Boolean / GF(2) product on B200 against the oracle
and the reference's golden vectors, bit-exact, for every kernel."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

GF2, BOOL = 1, 0
pytestmark = pytest.mark.gpu

# LOP3 (integer ALU); tcgen05 kind::mxf4 persistent CTA pairs (the default)
KERNELS = [1, 2]


def _bm(bmm, oracle, rows, cols, seed):
    return bmm.BitMatrix(rows, cols, oracle.random(rows, cols, seed))


@pytest.mark.parametrize("kernel", KERNELS)
def test_small_shapes_match_reference_words(engine, oracle, golden, kernel):
    bmm = engine
    for c in golden["cubic_small"]:
        a = _bm(bmm, oracle, c["m"], c["k"], c["a_seed"])
        b = _bm(bmm, oracle, c["k"], c["n"], c["b_seed"])
        got = bmm.multiply_cubic(a, b, bmm.Semiring(c["ring"]), kernel=kernel)
        assert [f"{int(x):016x}" for x in got.words] == c["words"], (c["m"], c["k"], c["n"], c["ring"])


def test_kernel64_matches_reference_golden(engine, oracle, golden):
    """bmmgpu_kernel64 (K9) on the reference's 64 x 64 golden block and its identities
    (reference test_engine.cpp:86-112), and its per-call latency (one launch + sync)."""
    import time
    bmm = engine
    g = golden["kernel64"]
    a = oracle.random(64, 64, g["a_seed"])
    bt = oracle.transpose_blocks64(64, 64, oracle.random(64, 64, g["b_seed"]))
    assert [f"{int(x):016x}" for x in bmm.kernel64(a, bt, bmm.Semiring.Gf2XorAnd)] == g["gf2"]
    assert [f"{int(x):016x}" for x in bmm.kernel64(a, bt, bmm.Semiring.BooleanOrAnd)] == g["bool"]
    ident = np.array([1 << i for i in range(64)], dtype=np.uint64)
    assert np.array_equal(bmm.kernel64(ident, bt, bmm.Semiring.Gf2XorAnd), oracle.random(64, 64, g["b_seed"]))
    ones = np.full(64, ~np.uint64(0), dtype=np.uint64)
    assert not bmm.kernel64(ones, ones, bmm.Semiring.Gf2XorAnd).any()
    assert np.all(bmm.kernel64(ones, ones, bmm.Semiring.BooleanOrAnd) == ~np.uint64(0))
    rng = np.random.default_rng(5)
    for _ in range(20):
        x = rng.integers(0, 2**63, 64, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 64, dtype=np.uint64)
        y = rng.integers(0, 2**63, 64, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 64, dtype=np.uint64)
        for ring in (GF2, BOOL):
            assert np.array_equal(bmm.kernel64(x, y, bmm.Semiring(ring)), oracle.kernel64(x, y, ring))
    lib = bmm.lib()
    out = np.zeros(64, dtype=np.uint64)
    reps = 2000
    t0 = time.perf_counter()
    for _ in range(reps):
        assert lib.bmmgpu_kernel64(a.ctypes.data, bt.ctypes.data, out.ctypes.data, GF2) == 0
    us = (time.perf_counter() - t0) / reps * 1e6
    print(f"bmmgpu_kernel64: {us:.1f} us per call")
    assert us < 200, us


@pytest.mark.parametrize("kernel", KERNELS)
def test_large_digests(engine, oracle, golden, kernel):
    bmm = engine
    for c in golden["cubic_large"]:
        a = _bm(bmm, oracle, c["m"], c["k"], c["a_seed"])
        b = _bm(bmm, oracle, c["k"], c["n"], c["b_seed"])
        got = bmm.multiply_cubic(a, b, bmm.Semiring(c["ring"]), kernel=kernel)
        assert f"{oracle.fnv1a64(got.words):016x}" == c["fnv"], c
        assert oracle.popcount(got.words) == c["pop"]


@pytest.mark.parametrize("kernel", KERNELS)
def test_sparse_boolean_is_not_vacuous(engine, oracle, golden, kernel):
    """Dense inputs make the Boolean product all ones; AND-of-k inputs do not."""
    bmm = engine
    for c in golden["sparse"]:
        n, k = c["n"], c["k"]
        a = np.full(n * n // 64, ~np.uint64(0), dtype=np.uint64)
        b = a.copy()
        for i in range(k):
            a &= oracle.random(n, n, 1 + 1000 * i)
            b &= oracle.random(n, n, 2 + 1000 * i)
        assert f"{oracle.fnv1a64(a):016x}" == c["a_fnv"]
        got = bmm.multiply_cubic(bmm.BitMatrix(n, n, a), bmm.BitMatrix(n, n, b), bmm.Semiring(c["ring"]),
                                 kernel=kernel)
        assert f"{oracle.fnv1a64(got.words):016x}" == c["fnv"], c
        assert oracle.popcount(got.words) == c["pop"]


@pytest.mark.parametrize("kernel", KERNELS)
def test_random_shapes_against_oracle(engine, oracle, kernel):
    bmm = engine
    rng = np.random.default_rng(11)
    shapes = [(1, 1, 1), (64, 64, 64), (63, 65, 127), (0, 5, 7), (5, 0, 7), (5, 7, 0), (1, 4097, 3),
              (300, 1025, 257), (129, 2048, 513), (64, 64, 1000), (1000, 64, 64)]
    shapes += [tuple(int(x) for x in rng.integers(1, 700, size=3)) for _ in range(12)]
    for t, (m, k, n) in enumerate(shapes):
        a = _bm(bmm, oracle, m, k, 300 + t)
        b = _bm(bmm, oracle, k, n, 400 + t)
        for ring in (GF2, BOOL):
            got = bmm.multiply_cubic(a, b, bmm.Semiring(ring), kernel=kernel)
            want = oracle.multiply_cubic(a.words, b.words, m, k, n, ring)
            assert np.array_equal(got.words, want), (m, k, n, ring)


@pytest.mark.parametrize("kernel", KERNELS)
def test_identity_all_ones_and_worked_example(engine, oracle, kernel):
    bmm = engine
    # 2x2 example (reference test_engine.cpp:114-131)
    a2, b2 = bmm.BitMatrix.zeros(2, 2), bmm.BitMatrix.zeros(2, 2)
    a2.set(0, 0, True); a2.set(0, 1, True); a2.set(1, 1, True)
    b2.set(0, 0, True); b2.set(1, 0, True); b2.set(1, 1, True)
    c = bmm.multiply_cubic(a2, b2, bmm.Semiring.Gf2XorAnd, kernel=kernel)
    assert [c.get(0, 0), c.get(0, 1), c.get(1, 0), c.get(1, 1)] == [False, True, True, True]
    c = bmm.multiply_cubic(a2, b2, bmm.Semiring.BooleanOrAnd, kernel=kernel)
    assert all(c.get(i, j) for i in range(2) for j in range(2))
    for ring in (bmm.Semiring.Gf2XorAnd, bmm.Semiring.BooleanOrAnd):
        ident = bmm.BitMatrix.zeros(128, 128)
        for i in range(128):
            ident.set(i, i, True)
        m = _bm(bmm, oracle, 128, 128, 21)
        assert bmm.multiply_cubic(ident, m, ring, kernel=kernel) == m
        assert bmm.multiply_cubic(m, ident, ring, kernel=kernel) == m
    ones = bmm.BitMatrix(256, 256, np.full(256 * 4, ~np.uint64(0), dtype=np.uint64))
    assert not bmm.multiply_cubic(ones, ones, bmm.Semiring.Gf2XorAnd, kernel=kernel).words.any()
    assert np.all(bmm.multiply_cubic(ones, ones, bmm.Semiring.BooleanOrAnd, kernel=kernel).words == ~np.uint64(0))


@pytest.mark.parametrize("kernel", KERNELS)
def test_accumulate_folds_partials(engine, oracle, kernel):
    """K-split integration: C = A[:, :k1] B[:k1] (+) A[:, k1:] B[k1:] (XOR / OR)."""
    bmm = engine
    m, k, n, k1 = 256, 2048, 512, 1024
    a = _bm(bmm, oracle, m, k, 71)
    b = _bm(bmm, oracle, k, n, 72)
    aw = a.words.reshape(m, k // 64)
    for ring in (GF2, BOOL):
        want = oracle.multiply_cubic(a.words, b.words, m, k, n, ring)
        a1 = bmm.BitMatrix(m, k1, np.ascontiguousarray(aw[:, :k1 // 64]).ravel())
        a2 = bmm.BitMatrix(m, k - k1, np.ascontiguousarray(aw[:, k1 // 64:]).ravel())
        b1 = bmm.BitMatrix(k1, n, b.words[: k1 * n // 64].copy())
        b2 = bmm.BitMatrix(k - k1, n, b.words[k1 * n // 64:].copy())
        c = bmm.multiply_cubic(a1, b1, bmm.Semiring(ring), kernel=kernel)
        bmm.multiply_cubic(a2, b2, bmm.Semiring(ring), kernel=kernel, out=c, accumulate=True)
        assert np.array_equal(c.words, want)


def test_device_api_panels(engine, oracle):
    """bmmgpu_dev_transpose + bmmgpu_dev_cubic on torch-owned HBM buffers."""
    import torch
    bmm = engine
    lib = bmm.lib()
    for kernel in KERNELS:
        gm, gn, gk = bmm.granularity(kernel)
        m, k, n = 300, 3000, 700
        a = oracle.random(m, k, 5)
        b = oracle.random(k, n, 6)
        m_pad, n_pad = -(-m // gm) * gm, -(-n // gn) * gn
        kw = -(-k // gk) * gk // 64
        dA = torch.zeros((m_pad, kw), dtype=torch.int64, device="cuda")
        dA[:m, : (k + 63) // 64] = torch.from_numpy(a.view(np.int64).reshape(m, -1)).cuda()
        dB = torch.from_numpy(b.view(np.int64)).cuda()
        dBt = torch.empty((n_pad, kw), dtype=torch.int64, device="cuda")
        dC = torch.empty((m_pad, n_pad // 64), dtype=torch.int64, device="cuda")
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        assert lib.bmmgpu_dev_transpose(dB.data_ptr(), (n + 63) // 64, k, n, dBt.data_ptr(), n_pad, kw, stream) == 0
        for ring in (GF2, BOOL):
            assert lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dBt.data_ptr(), kw, dC.data_ptr(), n_pad // 64, m_pad,
                                        n_pad, kw, ring, kernel, 0, stream) == 0
            torch.cuda.synchronize()
            got = dC.cpu().numpy().view(np.uint64)[:m, : (n + 63) // 64].ravel()
            assert np.array_equal(got, oracle.multiply_cubic(a, b, m, k, n, ring))


def test_rejects_bad_panels(engine):
    bmm = engine
    lib = bmm.lib()
    assert lib.bmmgpu_dev_cubic(None, 16, None, 16, None, 4, 65, 256, 16, 1, 1, 0, None) == 1
    assert b"m_pad" in lib.bmmgpu_last_error()


@pytest.mark.parametrize("mode,budget", [(1, 0), (1, 3 << 20), (1, 1 << 20), (1, 600 << 10), (2, 0), (2, 2 << 20)])
def test_out_of_core_streamed_driver(engine, oracle, mode, budget):
    """csrc/stream.cu: resident A panels, B streamed in double-buffered K-chunks,
    partial products folded on device -- bit-exact for every tiling the budget forces."""
    bmm = engine
    for (m, k, n) in [(1000, 5000, 700), (300, 2048, 1300), (64, 9000, 64)]:
        a = _bm(bmm, oracle, m, k, 81)
        b = _bm(bmm, oracle, k, n, 82)
        for ring in (GF2, BOOL):
            want = oracle.multiply_cubic(a.words, b.words, m, k, n, ring)
            got = bmm.multiply_cubic(a, b, bmm.Semiring(ring), force_streaming=mode, device_budget=budget)
            assert np.array_equal(got.words, want), (m, k, n, ring, budget)
            # accumulate through the streamed path: C (+)= A.B twice gives 0 (GF2) / the product (Boolean)
            bmm.multiply_cubic(a, b, bmm.Semiring(ring), out=got, accumulate=True, force_streaming=mode,
                               device_budget=budget)
            if ring == GF2:
                assert not got.words.any()
            else:
                assert np.array_equal(got.words, want)


@pytest.mark.parametrize("loader", ["tma", "cpasync"])
def test_umma_pair_loaders(engine, oracle, monkeypatch, loader):
    """The persistent pair kernel's two packed-bit loaders (TMA boxes / cp.async warps),
    including K tails that end inside a 4-stage superstage (TMA zero-fills past K)."""
    bmm = engine
    monkeypatch.setenv("BMMGPU_UMMA_LOADER", loader)
    shapes = [(256, 1024, 256), (256, 1280, 256), (512, 4096 + 768, 300), (300, 2048 + 64, 700), (700, 1536, 513)]
    for t, (m, k, n) in enumerate(shapes):
        a = _bm(bmm, oracle, m, k, 900 + t)
        b = _bm(bmm, oracle, k, n, 950 + t)
        for ring in (GF2, BOOL):
            got = bmm.multiply_cubic(a, b, bmm.Semiring(ring), kernel=2)
            want = oracle.multiply_cubic(a.words, b.words, m, k, n, ring)
            assert np.array_equal(got.words, want), (loader, m, k, n, ring)


def test_device_api_batched(engine, oracle):
    """bmmgpu_dev_cubic_batched: independent products in one launch, each equal to the
    oracle's product of its own panels (the leaf layer of the fast recursion)."""
    import torch
    bmm = engine
    lib = bmm.lib()
    for kernel in KERNELS:
        gm, gn, gk = bmm.granularity(kernel)
        batch, L = 5, 512
        m_pad, n_pad, kw = -(-L // gm) * gm, -(-L // gn) * gn, -(-L // gk) * gk // 64
        As = [oracle.random(L, L, 200 + i) for i in range(batch)]
        Bs = [oracle.random(L, L, 300 + i) for i in range(batch)]
        dA = torch.zeros((batch, m_pad, kw), dtype=torch.int64, device="cuda")
        dBt = torch.zeros((batch, n_pad, kw), dtype=torch.int64, device="cuda")
        dC = torch.zeros((batch, m_pad, n_pad // 64), dtype=torch.int64, device="cuda")
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for i in range(batch):
            dA[i, :L, : L // 64] = torch.from_numpy(As[i].view(np.int64).reshape(L, -1)).cuda()
            dB = torch.from_numpy(Bs[i].view(np.int64)).cuda()
            assert lib.bmmgpu_dev_transpose(dB.data_ptr(), L // 64, L, L, dBt[i].data_ptr(), n_pad, kw,
                                            stream) == 0
        for ring in (GF2, BOOL):
            assert lib.bmmgpu_dev_cubic_batched(dA.data_ptr(), kw, m_pad * kw, dBt.data_ptr(), kw, n_pad * kw,
                                                dC.data_ptr(), n_pad // 64, m_pad * (n_pad // 64), batch, m_pad,
                                                n_pad, kw, ring, kernel, 0, stream) == 0
            torch.cuda.synchronize()
            for i in range(batch):
                got = dC[i].cpu().numpy().view(np.uint64)[:L, : L // 64].ravel()
                assert np.array_equal(got, oracle.multiply_cubic(As[i], Bs[i], L, L, L, ring)), (kernel, ring, i)


@pytest.mark.parametrize("kernel", KERNELS)
def test_inner_dimension_beyond_fp32_exact_range(engine, kernel):
    """K = 2^23 + 2^20 bits: counts up to ~9.4e6 exceed the 2^23 the tensor-core kernels
    keep exact in fp32, so the dispatcher folds K-chunks of 2^22 bits (the reference's
    XOR / OR fold of partial products).  A row i = ones on [0, K - 3i), B column j =
    ones on [0, K - 37j): count = K - max(3i, 37j), parity known in closed form; the
    last row of A is zero (Boolean zeros)."""
    bmm = engine
    m = n = 256
    K = (1 << 23) + (1 << 20)
    W = K // 64
    A = np.full((m, W), np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    for i in range(m):
        L = K - 3 * i if i < m - 1 else 0
        A[i, L // 64 + 1:] = 0
        if L // 64 < W:
            A[i, L // 64] = np.uint64((1 << (L % 64)) - 1)
    B = np.full((K, n // 64), np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    tail = 37 * n
    ks = np.arange(K - tail, K)
    cols = np.minimum(n, -(-(K - ks) // 37))  # columns j with 37 j < K - k
    bits = (np.arange(n)[None, :] < cols[:, None])
    B[K - tail:] = np.packbits(bits, axis=1, bitorder="little").view(np.uint64)
    i = np.arange(m)[:, None]
    j = np.arange(n)[None, :]
    count = np.where(i == m - 1, 0, K - np.maximum(3 * i, 37 * j))
    for ring in (GF2, BOOL):
        want_bits = (count % 2 == 1) if ring == GF2 else (count > 0)
        want = np.packbits(want_bits, axis=1, bitorder="little").view(np.uint64).ravel()
        got = bmm.multiply_cubic(bmm.BitMatrix(m, K, A.ravel()), bmm.BitMatrix(K, n, B.ravel()),
                                 bmm.Semiring(ring), kernel=kernel)
        assert np.array_equal(got.words, want), (kernel, ring)


@pytest.mark.parametrize("shape", [(2048, 8192, 131072), (1024, 8256, 66560)])
def test_pageable_host_buffers_are_staged(engine, oracle, shape):
    """Large pageable operands (the reference API's std::vector storage) go through the
    library's pinned staging slots: same bits as the call on page-locked buffers, and
    rows checked independently.  First shape: B 128 MiB and C 32 MiB, both directions
    staged; second: B is 65.5 MiB, a contiguous copy wider than a staging slot that is
    not a whole number of the 1 MiB rows it is reshaped into (the remainder path)."""
    import torch
    bmm = engine
    m, k, n = shape
    a = oracle.random(m, k, 301)
    b = oracle.random(k, n, 302)
    for ring in (GF2, BOOL):
        got = bmm.multiply_cubic(bmm.BitMatrix(m, k, a), bmm.BitMatrix(k, n, b), bmm.Semiring(ring))
        ha = torch.from_numpy(a.view(np.int64)).pin_memory()
        hb = torch.from_numpy(b.view(np.int64)).pin_memory()
        hc = torch.zeros(m * n // 64, dtype=torch.int64).pin_memory()
        pinned = bmm.multiply_cubic(bmm.BitMatrix(m, k, ha.numpy().view(np.uint64)),
                                    bmm.BitMatrix(k, n, hb.numpy().view(np.uint64)), bmm.Semiring(ring),
                                    out=bmm.BitMatrix(m, n, hc.numpy().view(np.uint64)))
        assert np.array_equal(got.words, pinned.words), ring
        B = b.reshape(k, -(-n // 64))
        for i in (0, 777, m - 1):
            bits = np.unpackbits(a.reshape(m, -(-k // 64))[i].view(np.uint8), bitorder="little")[:k]
            sel = B[np.flatnonzero(bits)]
            want = np.bitwise_xor.reduce(sel, axis=0) if ring == GF2 else np.bitwise_or.reduce(sel, axis=0)
            assert np.array_equal(got.words.reshape(m, -(-n // 64))[i], want), (ring, i)


def test_concurrent_long_k_products_on_one_device(engine, oracle):
    """Two host threads run wave-aligned (long-K) products on the same GPU at once: the
    second launch's CTA pairs are not all resident while the first runs, so its
    loaders' bounded wave wait must give up instead of deadlocking; both results stay
    exact."""
    import threading
    bmm = engine
    m, k, n = 2048, 32768, 2048  # 128 K-stages: wave alignment on
    ins = [(oracle.random(m, k, 401 + i), oracle.random(k, n, 501 + i)) for i in range(2)]
    outs = [None, None]

    def run(i):
        a, b = ins[i]
        outs[i] = bmm.multiply_cubic(bmm.BitMatrix(m, k, a), bmm.BitMatrix(k, n, b), bmm.Semiring.Gf2XorAnd)

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th)
    for i in range(2):
        a, b = ins[i]
        A = a.reshape(m, k // 64)
        B = b.reshape(k, n // 64)
        for r in (0, m - 1):
            bits = np.unpackbits(A[r].view(np.uint8), bitorder="little")[:k]
            want = np.bitwise_xor.reduce(B[np.flatnonzero(bits)], axis=0)
            assert np.array_equal(outs[i].words.reshape(m, n // 64)[r], want), (i, r)


@pytest.mark.parametrize("slices", [None, "1", "3"])
def test_in_core_row_slices(engine, oracle, monkeypatch, slices):
    """csrc/capi.cu in-core path: A / C row slices pipelined behind B's upload, the last
    slice ragged (m = 4100: 17 row tiles) and padded columns / K; accumulate folds into
    the uploaded C slice by slice.  Same bits for any slice count."""
    bmm = engine
    if slices:
        monkeypatch.setenv("BMMGPU_INCORE_SLICES", slices)
    m, k, n = 4100, 777, 1000
    a = _bm(bmm, oracle, m, k, 91)
    b = _bm(bmm, oracle, k, n, 92)
    for ring in (GF2, BOOL):
        want = oracle.multiply_cubic(a.words, b.words, m, k, n, ring)
        c = bmm.multiply_cubic(a, b, bmm.Semiring(ring))
        assert np.array_equal(c.words, want), ring
        bmm.multiply_cubic(a, b, bmm.Semiring(ring), out=c, accumulate=True)
        twice = np.zeros_like(want) if ring == GF2 else want
        assert np.array_equal(c.words, twice), ring


def test_concurrent_calls_lease_distinct_streams(engine, oracle):
    """Four host threads call the host API at once: each call leases its own streams
    from the per-device pool (csrc/capi.cu StreamSet), results stay exact, and repeated
    calls reuse the pooled streams."""
    import threading
    bmm = engine
    m = k = n = 4096
    ins = [(oracle.random(m, k, 601 + i), oracle.random(k, n, 701 + i)) for i in range(4)]
    wants = [oracle.multiply_cubic(a, b, m, k, n, GF2) for a, b in ins]
    outs = [None] * 4

    def run(i):
        a, b = ins[i]
        for _ in range(3):
            outs[i] = bmm.multiply_cubic(bmm.BitMatrix(m, k, a), bmm.BitMatrix(k, n, b), bmm.Semiring.Gf2XorAnd)

    th = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th)
    for i in range(4):
        assert np.array_equal(outs[i].words, wants[i]), i


@pytest.mark.parametrize("ring", [GF2, BOOL])
def test_wave_aligned_mode_matches_oracle(engine, oracle, ring):
    """The headline kernel mode: long-K products with more output tiles than CTA pairs run
    with wave-aligned TMA loaders and the L2 eviction policy (cubic_umma2.cu loader).
    4096 x 16384 x 4096 in core: 2 row slices of 128 tiles each over 74 pairs, 64 K-stages.
    The debug counters prove the mode ran and never hit its spin limit; the product is
    compared word for word with the oracle (Boolean on AND-of-7 inputs, ~63 % ones)."""
    bmm = engine
    lib = bmm.lib()
    m, k, n = 4096, 16384, 4096
    a = oracle.random(m, k, 601)
    b = oracle.random(k, n, 602)
    if ring == BOOL:
        for s in range(6):
            a &= oracle.random(m, k, 611 + s)
            b &= oracle.random(k, n, 621 + s)
    before, t_before = ctypes.c_uint64(), ctypes.c_uint64()
    assert lib.bmmgpu_debug_wave_stats(ctypes.byref(before), ctypes.byref(t_before)) == 0
    got = bmm.multiply_cubic(bmm.BitMatrix(m, k, a), bmm.BitMatrix(k, n, b), bmm.Semiring(ring))
    after, t_after = ctypes.c_uint64(), ctypes.c_uint64()
    assert lib.bmmgpu_debug_wave_stats(ctypes.byref(after), ctypes.byref(t_after)) == 0
    assert after.value > before.value, "wave alignment did not engage"
    assert t_after.value == t_before.value, "a loader gave up wave alignment"
    want = oracle.multiply_cubic(a, b, m, k, n, ring)
    assert np.array_equal(got.words, want)
    if ring == BOOL:
        frac = float(np.unpackbits(want.view(np.uint8)).mean())
        assert 0.3 < frac < 0.9, frac


@pytest.mark.parametrize("ring", [GF2, BOOL])
def test_tmem_operand_mode_matches_oracle(engine, oracle, ring):
    """Long-K launches keep operand A in tensor memory (kTs: tcgen05.mma with A from TMEM,
    one accumulator).  Through the device API, one launch each: 2560 x 32768 x 2048 (80 tiles
    over 74 pairs, 128 K-stages), 768 x 65536 x 512 (256 stages, fewer tiles than pairs) and
    512 x 33024 x 768 (129 stages: a partial superstage at the end of K), the second also with
    the accumulate flag (the K-chunk fold); the debug counter proves the
    mode ran; word for word against the oracle (Boolean on AND-of-7 inputs)."""
    import torch
    bmm = engine
    lib = bmm.lib()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for m, k, n, seed in ((2560, 32768, 2048, 701), (768, 65536, 512, 731), (512, 33024, 768, 761)):
        a = oracle.random(m, k, seed)
        b = oracle.random(k, n, seed + 1)
        if ring == BOOL:
            for s in range(6):
                a &= oracle.random(m, k, seed + 10 + s)
                b &= oracle.random(k, n, seed + 20 + s)
        kw, nw = k // 64, n // 64
        dA = torch.from_numpy(a.view(np.int64).reshape(m, kw)).cuda()
        dB = torch.from_numpy(b.view(np.int64).reshape(k, nw)).cuda()
        dBt = torch.empty((n, kw), dtype=torch.int64, device="cuda")
        dC = torch.empty((m, nw), dtype=torch.int64, device="cuda")
        assert lib.bmmgpu_dev_transpose(dB.data_ptr(), nw, k, n, dBt.data_ptr(), n, kw, stream) == 0
        before, after = ctypes.c_uint64(), ctypes.c_uint64()
        assert lib.bmmgpu_debug_ts_launches(ctypes.byref(before)) == 0
        assert lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dBt.data_ptr(), kw, dC.data_ptr(), nw, m, n, kw, ring, 2, 0,
                                    stream) == 0
        torch.cuda.synchronize()
        assert lib.bmmgpu_debug_ts_launches(ctypes.byref(after)) == 0
        assert after.value == before.value + 1, "the TMEM-operand mode did not run"
        want = oracle.multiply_cubic(a, b, m, k, n, ring)
        assert np.array_equal(dC.cpu().numpy().view(np.uint64).ravel(), want), (m, k, n)
        if k == 65536:
            c0 = oracle.random(m, n, seed + 5)
            dC.copy_(torch.from_numpy(c0.view(np.int64).reshape(m, nw)).cuda())
            assert lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dBt.data_ptr(), kw, dC.data_ptr(), nw, m, n, kw, ring, 2,
                                        1, stream) == 0
            torch.cuda.synchronize()
            folded = (c0 ^ want) if ring == GF2 else (c0 | want)
            assert np.array_equal(dC.cpu().numpy().view(np.uint64).ravel(), folded)
