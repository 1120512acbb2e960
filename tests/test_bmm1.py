"""BMM1 files (reference bitmatrix.cpp:187-233) through the C ABI's parallel reader /
writer: round trips against the reference's own writer and reader (oracle/_ref), the
reference's rejection cases and messages, and -- on the GPU box, where page-locked
memory exists -- a 4 GiB matrix read straight into pinned memory and multiplied."""
from __future__ import annotations

import os
import struct
import time

import numpy as np
import pytest

from conftest import HAS_GPU, ROOT


@pytest.fixture()
def bmm():
    import paper_1909_01554_b200 as m
    return m


def test_round_trip_and_reference_interop(bmm, oracle, tmp_path):
    from oracle import REF_SO, Reference
    for rows, cols, seed in [(1, 1, 1), (130, 130, 7), (64, 4096, 3), (300, 65, 9)]:
        m = bmm.BitMatrix(rows, cols, oracle.random(rows, cols, seed))
        p = tmp_path / f"m{rows}x{cols}.bmm"
        bmm.write_bmm1(m, p, threads=3)
        assert p.stat().st_size == 20 + 8 * m.words.size
        raw = p.read_bytes()
        assert raw[:4] == b"BMM1" and struct.unpack("<QQ", raw[4:20]) == (rows, cols)
        assert bmm.read_bmm1(p, threads=2) == m
        if REF_SO.exists():
            ref = Reference()
            r, c, w = ref.read_bmm1(str(p))
            assert (r, c) == (rows, cols) and np.array_equal(w, m.words)
            q = tmp_path / "ref.bmm"
            ref.write_bmm1(str(q), rows, cols, m.words)
            assert q.read_bytes() == raw and bmm.read_bmm1(q) == m


def test_rejects_malformed_files_like_the_reference(bmm, oracle, tmp_path):
    m = bmm.BitMatrix(3, 70, oracle.random(3, 70, 2))
    good = tmp_path / "good.bmm"
    bmm.write_bmm1(m, good)
    raw = good.read_bytes()
    cases = {
        "truncated header": raw[:10],
        "bad magic": b"BMM2" + raw[4:],
        "unreasonable dimensions": raw[:4] + struct.pack("<QQ", 0, 70) + raw[20:],
        "truncated payload": raw[:-8],
        "trailing bytes": raw + b"\0",
        "nonzero padding bits": raw[:20 + 8] + struct.pack("<Q", 1 << 63) + raw[20 + 16:],
    }
    for msg, data in cases.items():
        p = tmp_path / "bad.bmm"
        p.write_bytes(data)
        with pytest.raises(bmm.FormatError, match=msg):
            bmm.read_bmm1(p)
    with pytest.raises(bmm.FormatError, match="cannot open"):
        bmm.read_bmm1(tmp_path / "missing.bmm")


@pytest.mark.gpu
@pytest.mark.skipif(not HAS_GPU, reason="page-locked memory needs the CUDA driver")
def test_four_gib_matrix_into_pinned_memory(bmm, tmp_path):
    """A 262144 x 131072 matrix (4 GiB payload) written and read back with the parallel
    positioned I/O, the read going straight into page-locked memory; then one row panel of
    it is multiplied on the GPU from that memory and checked row-wise in numpy."""
    rows, cols = 262144, 131072
    n = rows * cols // 64
    src = bmm.PinnedWords(n)
    bmm.random_rows_into(src.words, cols, 5, 0, rows)
    p = tmp_path / "big.bmm"
    t0 = time.perf_counter()
    bmm.write_bmm1(bmm.BitMatrix(rows, cols, src.words), p)
    t_w = time.perf_counter() - t0
    dst = bmm.PinnedWords(n)
    t0 = time.perf_counter()
    m = bmm.read_bmm1(p, out=dst.words)
    t_r = time.perf_counter() - t0
    assert (m.rows, m.cols) == (rows, cols)
    assert np.array_equal(dst.words[:: 1 << 20], src.words[:: 1 << 20])
    assert np.array_equal(dst.words[-4096:], src.words[-4096:])
    assert bmm.lib().bmmgpu_last_error is not None
    print(f"BMM1 4 GiB: write {4 / t_w:.1f} GiB/s, read into pinned memory {4 / t_r:.1f} GiB/s")
    # A = rows [0, 256) of the file (256 x 131072), B = a 131072 x 256 slice of it transposed is
    # not needed: multiply A . M[0:131072, 0:256] on the GPU and check two rows in numpy
    a = bmm.BitMatrix(256, cols, m.words[: 256 * (cols // 64)])
    bw = cols // 64
    bsub = np.ascontiguousarray(m.words.reshape(rows, bw)[:cols, :4]).ravel()
    b = bmm.BitMatrix(cols, 256, bsub)
    c = bmm.multiply_cubic(a, b, bmm.Semiring.Gf2XorAnd)
    B = bsub.reshape(cols, 4)
    for i in (0, 255):
        bits = np.unpackbits(a.words.reshape(256, bw)[i].view(np.uint8), bitorder="little")
        want = np.bitwise_xor.reduce(B[np.flatnonzero(bits)], axis=0)
        assert np.array_equal(c.words.reshape(256, 4)[i], want)
    os.unlink(p)
    src.free()
    dst.free()
