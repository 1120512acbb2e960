"""CPU: pin the C restatement (oracle/) against the reference's golden vectors
and, where oracle/_ref is built, against the reference itself."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import REF_SO, REF_SRC

GF2, BOOL = 1, 0


def test_mt19937_64_known_answer(oracle, golden):
    kat = golden["mt64_kat"]
    assert oracle.mt64(kat["seed"], kat["index"])[-1] == int(kat["value"]) == 9981545732273789042


def test_random_matches_reference_digests(oracle, golden):
    for r in golden["random"]:
        w = oracle.random(r["rows"], r["cols"], r["seed"])
        assert f"{oracle.fnv1a64(w):016x}" == r["fnv"], r
        assert oracle.popcount(w) == r["pop"]
        assert f"{int(w[0]):016x}" == r["w0"]


def test_random_is_pad_clean_and_dense(oracle):
    w = oracle.random(130, 130, 3).reshape(130, 3)
    assert not np.any(w[:, 2] & ~np.uint64((1 << 2) - 1))
    for seed in range(4):
        d = oracle.popcount(oracle.random(1024, 1024, seed)) / 1024**2
        assert 0.45 < d < 0.55


def test_kernel64(oracle, golden):
    g = golden["kernel64"]
    a = oracle.random(64, 64, g["a_seed"])
    bt = oracle.transpose_blocks64(64, 64, oracle.random(64, 64, g["b_seed"]))
    assert [f"{int(x):016x}" for x in oracle.kernel64(a, bt, GF2)] == g["gf2"]
    assert [f"{int(x):016x}" for x in oracle.kernel64(a, bt, BOOL)] == g["bool"]
    ident = np.array([1 << i for i in range(64)], dtype=np.uint64)
    b = oracle.random(64, 64, g["b_seed"])
    assert np.array_equal(oracle.kernel64(ident, bt, GF2), b)
    ones = np.full(64, ~np.uint64(0), dtype=np.uint64)
    assert not oracle.kernel64(ones, ones, GF2).any()
    assert np.all(oracle.kernel64(ones, ones, BOOL) == ~np.uint64(0))


def test_cubic_small_full_words(oracle, golden):
    for c in golden["cubic_small"]:
        a = oracle.random(c["m"], c["k"], c["a_seed"])
        b = oracle.random(c["k"], c["n"], c["b_seed"])
        got = oracle.multiply_cubic(a, b, c["m"], c["k"], c["n"], c["ring"])
        assert [f"{int(x):016x}" for x in got] == c["words"], (c["m"], c["k"], c["n"], c["ring"])


@pytest.mark.parametrize("idx", range(8))
def test_cubic_large_digests(oracle, golden, idx):
    c = golden["cubic_large"][idx]
    if c["m"] * c["k"] * c["n"] > 4096**3:
        pytest.skip("n=8192 is checked on the GPU against the same digest")
    a = oracle.random(c["m"], c["k"], c["a_seed"])
    b = oracle.random(c["k"], c["n"], c["b_seed"])
    got = oracle.multiply_cubic(a, b, c["m"], c["k"], c["n"], c["ring"])
    assert f"{oracle.fnv1a64(got):016x}" == c["fnv"]
    assert oracle.popcount(got) == c["pop"]


def test_interleave_digests(oracle, golden):
    for c in golden["interleave"]:
        n = 64 << c["depth"]
        m = oracle.random(n, n, c["seed"])
        t = oracle.to_interleaved(c["depth"], c["which"], m)
        assert f"{oracle.fnv1a64(t):016x}" == c["fnv"], c
        assert np.array_equal(oracle.from_interleaved(c["depth"], c["which"], t), m)


def test_interleave_worked_example(oracle):
    # test_bitmatrix.cpp:151-164
    assert oracle.interleaved_bit_index(1, 0, 66, 5) == 2 * 4096 + 2 * 64 + 5
    assert oracle.interleaved_bit_index(1, 1, 66, 5) == 2 * 4096 + 5 * 64 + 2
    assert oracle.interleaved_bit_index(1, 2, 66, 5) == 2 * 4096 + 2 * 64 + 5


def test_basis_change_alt_si(oracle, golden):
    v = oracle.random(1, 4 * 4 * 4096, 41)
    for c in golden["basis_change"]:
        if c["scheme"] != 1:
            continue  # the C restatement carries the alt-si constants only
        which = c["which"]
        out = oracle.basis_change(v, 2, which)
        assert f"{oracle.fnv1a64(out):016x}" == c["fnv"], c
        assert np.array_equal(oracle.basis_change(out, 2, which), v)  # self-inverse


def test_multiply_alt_on_hat_vectors(oracle, golden):
    for c in golden["multiply_alt"]:
        if c["scheme"] != 1:  # the oracle restates the alt-si scheme; the GPU test covers all three
            continue
        depth = c["d_serial"] + c["d_parallel"]
        n = 64 << depth
        ah = oracle.random(1, n * n, c["a_seed"])
        bh = oracle.random(1, n * n, c["b_seed"])
        got = oracle.multiply_alt(ah, bh, depth)
        assert f"{oracle.fnv1a64(got):016x}" == c["fnv"], c


def test_alt_si_full_product(oracle, golden):
    for c in golden["fast"]:
        if c["algo"] != 2 or c["n"] > 1024:
            continue
        n = c["n"]
        depth = (n // 64).bit_length() - 1
        a, b = oracle.random(n, n, c["a_seed"]), oracle.random(n, n, c["b_seed"])
        got = oracle.multiply_alt_si(a, b, depth)
        assert f"{oracle.fnv1a64(got):016x}" == c["fnv"], c
        assert np.array_equal(got, oracle.multiply_cubic(a, b, n, n, n, GF2))


@pytest.mark.skipif(not (REF_SO.exists() or REF_SRC.exists()), reason="reference not available here")
def test_oracle_matches_reference_on_random_shapes(oracle):
    from oracle import Reference
    ref = Reference()
    rng = np.random.default_rng(7)
    for trial in range(30):
        m, k, n = (int(x) for x in rng.integers(1, 300, size=3))
        if trial % 3 == 0:
            m, k, n = 64 * int(rng.integers(1, 4)), 64 * int(rng.integers(1, 4)), 64 * int(rng.integers(1, 4))
        a, b = ref.random(m, k, 100 + trial), ref.random(k, n, 200 + trial)
        assert np.array_equal(a, oracle.random(m, k, 100 + trial))
        for ring in (GF2, BOOL):
            assert np.array_equal(oracle.multiply_cubic(a, b, m, k, n, ring),
                                  ref.multiply_cubic(a, b, m, k, n, ring)), (m, k, n, ring)
    for depth in (0, 1, 2, 3):
        n = 64 << depth
        a, b = ref.random(n, n, 5 + depth), ref.random(n, n, 6 + depth)
        assert np.array_equal(oracle.multiply_alt_si(a, b, depth),
                              ref.multiply(a, b, n, 2, 0, depth, 0, 1, GF2))
        for which in (0, 1, 2):
            t = ref.to_interleaved(depth, which, a)
            assert np.array_equal(t, oracle.to_interleaved(depth, which, a))
            assert np.array_equal(ref.basis_change(t, depth, which, 1), oracle.basis_change(t, depth, which))
