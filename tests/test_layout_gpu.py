"""Layout conversions on the GPU (csrc/layout.cu, bmmgpu_layout): transpose_blocks64,
to_interleaved, from_interleaved (reference bitmatrix.cpp:97-173), against the reference's
digests (tests/golden, made by oracle/_ref) and the oracle, through the device path and the
host-streamed path with small forced super-tiles, from pageable and page-locked buffers."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_interleave_matches_reference_digests(engine, oracle, golden):
    for c in golden["interleave"]:
        n = 64 << c["depth"]
        plan = engine.LayerPlan(0, 0, c["depth"], 1, 1)
        m = engine.BitMatrix(n, n, oracle.random(n, n, c["seed"]))
        t = engine.to_interleaved(m, plan, engine.Operand(c["which"]))
        assert f"{oracle.fnv1a64(t):016x}" == c["fnv"], c
        assert int(t[0]) == int(c["w0"], 16)
        assert engine.from_interleaved(t, plan, engine.Operand(c["which"])) == m


@pytest.mark.parametrize("piece", [None, "64", "128", "512"])
@pytest.mark.parametrize("depth", [0, 3, 6])
def test_streamed_interleave_equals_oracle(engine, oracle, monkeypatch, piece, depth):
    if piece:
        monkeypatch.setenv("BMMGPU_LAYOUT_PIECE", piece)
    n = 64 << depth
    plan = engine.LayerPlan(0, depth, 0, 1, 1)
    m = oracle.random(n, n, 1000 + depth)
    for which in (0, 1, 2):
        want = oracle.to_interleaved(depth, which, m)
        got = engine.to_interleaved(engine.BitMatrix(n, n, m), plan, engine.Operand(which))
        assert np.array_equal(got, want), (piece, depth, which)
        back = engine.from_interleaved(want, plan, engine.Operand(which))
        assert np.array_equal(back.words, m), (piece, depth, which)


@pytest.mark.parametrize("rows,cols", [(64, 64), (128, 640), (1984, 128), (4096, 4096), (192, 8192)])
def test_transpose_blocks64_equals_oracle(engine, oracle, rows, cols):
    w = oracle.random(rows, cols, rows + cols)
    want = oracle.transpose_blocks64(rows, cols, w)
    m = engine.BitMatrix(rows, cols, w.copy())
    engine.transpose_blocks64(m)
    assert np.array_equal(m.words, want)
    engine.transpose_blocks64(m)
    assert np.array_equal(m.words, w)


def test_layout_shape_errors(engine):
    with pytest.raises(engine.ShapeError):
        engine.transpose_blocks64(engine.BitMatrix.zeros(64, 100))
    with pytest.raises(engine.ShapeError):
        engine.to_interleaved(engine.BitMatrix.zeros(64, 64), engine.LayerPlan(0, 0, 1, 1, 1), engine.Operand.Left)
    w = np.zeros(96 * 2, dtype=np.uint64)
    with pytest.raises(engine.ShapeError):  # interleave needs n = 64 * 2^d
        engine.layout(w, w.copy(), 96, 96, engine.LAYOUT_TO_INTERLEAVED)
    with pytest.raises(ValueError):  # interleave is out of place
        engine.layout(w, w, 64, 64, engine.LAYOUT_TO_INTERLEAVED)


def test_device_layout_round_trip(engine, oracle):
    import ctypes

    import torch
    n, depth = 2048, 5
    m = oracle.random(n, n, 5)
    d = torch.from_numpy(m.view(np.int64)).cuda()
    t = torch.empty_like(d)
    back = torch.empty_like(d)
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    L = engine.lib()
    assert L.bmmgpu_dev_layout(d.data_ptr(), t.data_ptr(), n, n, engine.LAYOUT_TO_INTERLEAVED_RIGHT, sp) == 0
    assert L.bmmgpu_dev_layout(t.data_ptr(), back.data_ptr(), n, n, engine.LAYOUT_FROM_INTERLEAVED_RIGHT, sp) == 0
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy().view(np.uint64), oracle.to_interleaved(depth, 1, m))
    assert np.array_equal(back.cpu().numpy().view(np.uint64), m)


def test_large_pinned_round_trip_and_spot_blocks(engine, oracle):
    """n = 32768 (128 MiB per matrix) from page-locked buffers: several super-tiles per
    side; to -> from is the identity, blocks at the corners and the middle are checked
    against the reference's block map, and transpose_blocks64 twice is the identity."""
    n, depth = 32768, 9
    plan = engine.LayerPlan(0, 0, depth, 1, 1)
    src = engine.PinnedWords(n * n // 64)
    vec = engine.PinnedWords(n * n // 64)
    dst = engine.PinnedWords(n * n // 64)
    try:
        rng = np.random.default_rng(3)
        src.words[:] = rng.integers(0, 2**63, size=src.words.size, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
        engine.to_interleaved(engine.BitMatrix(n, n, src.words), plan, engine.Operand.Right, out=vec.words)
        w = n // 64
        for bi, bj in [(0, 0), (0, w - 1), (w - 1, 0), (w - 1, w - 1), (w // 2 + 3, w // 3)]:
            blk = src.words.reshape(n, w)[64 * bi:64 * bi + 64, bj].copy()
            want = oracle.transpose_blocks64(64, 64, blk)
            mb = oracle.interleaved_bit_index(depth, 1, 64 * bi, 64 * bj) // 64
            assert np.array_equal(vec.words[mb:mb + 64], want), (bi, bj)
        engine.from_interleaved(vec.words, plan, engine.Operand.Right, out=dst.words)
        assert np.array_equal(dst.words, src.words)
        m = engine.BitMatrix(n, n, dst.words)
        engine.transpose_blocks64(m)
        assert not np.array_equal(dst.words[:64], src.words[:64])
        engine.transpose_blocks64(m)
        assert np.array_equal(dst.words, src.words)
    finally:
        src.free()
        vec.free()
        dst.free()
