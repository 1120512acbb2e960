"""The bench's at-size parity checkers (bench.py) are themselves checked here on CPU
against the oracle: the GF(2) matrix x 64-column product used by Freivalds, Freivalds
accepting the true product and rejecting single-bit corruptions, and the numpy row /
column recomputation."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import bench


@pytest.mark.parametrize("m,k", [(64, 64), (200, 136), (512, 1000)])
def test_gf2_matvec64_matches_oracle(oracle, m, k):
    a = oracle.random(m, k, 5)
    x = oracle.random(k, 64, 6)  # k rows of one word: 64 bit-columns
    y = bench.gf2_matvec64(torch.from_numpy(a.view(np.int64)).view(m, -1), k, torch.from_numpy(x.view(np.int64)))
    assert np.array_equal(y.numpy().view(np.uint64), oracle.multiply_cubic(a, x, m, k, 64, 1))


@pytest.mark.parametrize("ring", [1, 0])
def test_freivalds_and_numpy_rows_accept_truth_and_reject_flips(oracle, ring):
    m = k = n = 512
    a = oracle.random(m, k, 1)
    b = oracle.random(k, n, 2)
    c = oracle.multiply_cubic(a, b, m, k, n, ring)
    T = lambda w, r: torch.from_numpy(w.view(np.int64)).view(r, -1)  # noqa: E731
    w = n // 64
    if ring == 1:
        assert bench.freivalds_gf2(T(a, m), T(b, k), T(c, m), m, k, n)
    assert bench.spot_check(a, b, c, n, ring, [0, 77, m - 1], 300, m)
    for (i, j) in [(0, 0), (77, 300), (m - 1, n - 1)]:
        bad = c.copy()
        bad[i * w + j // 64] ^= np.uint64(1) << np.uint64(j % 64)
        if ring == 1:
            assert not bench.freivalds_gf2(T(a, m), T(b, k), T(bad, m), m, k, n)
        assert not bench.spot_check(a, b, bad, n, ring, [i], j, m)


def test_reference_arm_without_the_reference_prints_unavailable(monkeypatch, capsys):
    """`bench.py --impl reference` on a box where oracle/_ref is missing (and the reference
    sources absent) must still print its one JSON line -- {"impl": "reference",
    "unavailable": ...} -- and return normally, not crash the driver's run."""
    import json
    import sys
    from pathlib import Path
    import oracle
    monkeypatch.setattr(oracle, "REF_SO", Path("/nonexistent/libbmmref.so"))
    monkeypatch.setattr(oracle, "REF_SRC", Path("/nonexistent/proj"))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"])
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    bench.main()
    lines = [ln for ln in capsys.readouterr().out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and "unavailable" in rec
