"""Generate tests/golden/golden.json from the UNMODIFIED reference.

Runs oracle/_ref/libbmmref.so (reference bmm_core compiled from
/root/reference/proj/src by oracle/Makefile) and records digests (FNV-1a 64
over the LE bytes of the word array, popcount, first word) or full word lists
for small cases.  Re-run with:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import Oracle, Reference  # noqa: E402

GF2, BOOL = 1, 0
OUT = Path(__file__).resolve().parent / "golden.json"


def hexw(w: np.ndarray) -> list[str]:
    return [f"{int(x):016x}" for x in w]


def main() -> None:
    ref = Reference()
    orc = Oracle()  # only for the FNV helper
    workers = os.cpu_count() or 1
    g: dict = {"generator": "tests/golden/make_golden.py via oracle/_ref (reference bmm_core)", "cases": {}}
    C = g["cases"]

    def digest(w: np.ndarray) -> dict:
        return {"fnv": f"{orc.fnv1a64(w):016x}", "pop": orc.popcount(w), "w0": f"{int(w[0]):016x}" if w.size else ""}

    # std::mt19937_64 known answer: 10000th draw of seed 5489 ([rand.predef])
    row = ref.random(1, 64 * 10000, 5489)
    C["mt64_kat"] = {"seed": 5489, "index": 10000, "value": str(int(row[-1]))}

    # generators
    C["random"] = []
    for rows, cols, seed in [(130, 130, 7), (130, 130, 3), (100, 200, 42), (64, 64, 5), (1024, 1024, 0),
                             (8192, 8192, 1), (8192, 8192, 2), (4096, 4096, 1), (4096, 4096, 2)]:
        w = ref.random(rows, cols, seed)
        C["random"].append({"rows": rows, "cols": cols, "seed": seed, **digest(w)})

    # kernel64 (test_engine.cpp:86-112 inputs)
    a = ref.random(64, 64, 11)
    bt = ref.transpose_blocks64(64, 64, ref.random(64, 64, 12))
    C["kernel64"] = {"a_seed": 11, "b_seed": 12, "gf2": hexw(ref.kernel64(a, bt, GF2)),
                     "bool": hexw(ref.kernel64(a, bt, BOOL))}

    # small cubic products, full outputs (test_engine.cpp:114-151 shapes)
    C["cubic_small"] = []
    for m, k, n, sa, sb in [(128, 192, 64, 22, 23), (130, 70, 50, 24, 25), (128, 128, 128, 51, 52),
                            (64, 64, 64, 11, 12), (1, 1, 1, 3, 4), (65, 129, 63, 5, 6), (200, 64, 300, 7, 8),
                            (64, 1000, 64, 9, 10), (3, 5, 700, 13, 14)]:
        A, B = ref.random(m, k, sa), ref.random(k, n, sb)
        for ring in (GF2, BOOL):
            c = ref.multiply_cubic(A, B, m, k, n, ring, workers)
            C["cubic_small"].append({"m": m, "k": k, "n": n, "a_seed": sa, "b_seed": sb, "ring": ring,
                                     "words": hexw(c)})

    # larger cubic products, digests
    C["cubic_large"] = []
    t0 = time.time()
    for m, k, n, sa, sb in [(4096, 4096, 4096, 1, 2), (8192, 8192, 8192, 1, 2), (1000, 3000, 500, 31, 32),
                            (2048, 8192, 1024, 33, 34)]:
        A, B = ref.random(m, k, sa), ref.random(k, n, sb)
        for ring in (GF2, BOOL):
            c = ref.multiply_cubic(A, B, m, k, n, ring, workers)
            C["cubic_large"].append({"m": m, "k": k, "n": n, "a_seed": sa, "b_seed": sb, "ring": ring,
                                     **digest(c)})
    print("cubic_large", time.time() - t0, "s", flush=True)

    # sparse Boolean parity inputs: AND of k seeded matrices
    C["sparse"] = []
    for n, kk in [(8192, 7), (2048, 5)]:
        A = np.full(n * n // 64, ~np.uint64(0), dtype=np.uint64)
        B = A.copy()
        for i in range(kk):
            A &= ref.random(n, n, 1 + 1000 * i)
            B &= ref.random(n, n, 2 + 1000 * i)
        for ring in (GF2, BOOL):
            c = ref.multiply_cubic(A, B, n, n, n, ring, workers)
            C["sparse"].append({"n": n, "k": kk, "a_seeds": "1+1000i", "b_seeds": "2+1000i", "ring": ring,
                                **digest(c), "a_fnv": f"{orc.fnv1a64(A):016x}"})

    # fast algorithms through the reference multiply(); algo 1 sw, 2 alt-si, 3 alt-chain
    C["fast"] = []
    for n, sa, sb, algo, plan in [(256, 53, 54, 2, (0, 2, 0)), (256, 53, 54, 2, (0, 1, 1)), (256, 53, 54, 2, (0, 0, 2)),
                                  (128, 93, 94, 1, (0, 0, 1)), (128, 93, 94, 3, (0, 1, 0)),
                                  (1024, 61, 62, 2, (0, 1, 3)), (4096, 1, 2, 2, (0, 3, 3)),
                                  (2048, 71, 72, 3, (0, 2, 3)), (2048, 71, 72, 1, (0, 2, 3))]:
        A, B = ref.random(n, n, sa), ref.random(n, n, sb)
        c, cnt = ref.multiply(A, B, n, algo, *plan, workers=1, ring=GF2, counts=True)
        C["fast"].append({"n": n, "a_seed": sa, "b_seed": sb, "algo": algo, "plan": list(plan), **digest(c),
                          "counts": [int(x) for x in cnt]})

    # interleave and basis change (test_bitmatrix.cpp:151-226, test_engine.cpp:226-289)
    C["interleave"] = []
    for depth in (0, 1, 2, 3):
        n = 64 << depth
        m = ref.random(n, n, 77 + depth)
        for which in (0, 1, 2):
            t = ref.to_interleaved(depth, which, m)
            C["interleave"].append({"depth": depth, "seed": 77 + depth, "which": which, **digest(t)})
    v = ref.random(1, 4 * 4 * 4096, 41)
    C["basis_change"] = []
    for scheme in (1, 2):  # AltSelfInverse, AltChaining (bmm::Builtin order)
        for which in (0, 1, 2):
            out = ref.basis_change(v, 2, which, scheme)
            C["basis_change"].append({"levels": 2, "seed": 41, "scheme": scheme, "which": which, **digest(out)})

    # multiply_alt on random hat vectors (test_engine.cpp:312-357)
    C["multiply_alt"] = []
    for ds, dp, sa, sb in [(1, 1, 63, 65), (2, 1, 61, 62), (0, 3, 71, 72)]:
        depth = ds + dp
        n = 64 << depth
        ah = ref.random(1, n * n, sa)
        bh = ref.random(1, n * n, sb)
        c = ref.multiply_alt(ah, bh, ds, dp, 1, 1)
        C["multiply_alt"].append({"d_serial": ds, "d_parallel": dp, "a_seed": sa, "b_seed": sb, "scheme": 1,
                                  **digest(c)})
    # the other two schemes, and a deeper alt-si vector (n = 2048) for the GPU tests
    for scheme, ds, dp, sa, sb in [(0, 1, 2, 81, 82), (2, 1, 2, 83, 84), (1, 2, 3, 85, 86)]:
        depth = ds + dp
        n = 64 << depth
        ah = ref.random(1, n * n, sa)
        bh = ref.random(1, n * n, sb)
        c = ref.multiply_alt(ah, bh, ds, dp, 1, scheme)
        C["multiply_alt"].append({"d_serial": ds, "d_parallel": dp, "a_seed": sa, "b_seed": sb, "scheme": scheme,
                                  **digest(c)})

    # pipeline::coordinate (the host layer) on hat vectors: outputs and op counts
    C["coordinate"] = []
    for scheme, dh, ds, dp, sa, sb, workers in [(1, 1, 1, 1, 91, 92, 2), (1, 2, 0, 1, 93, 94, 3),
                                                (2, 2, 1, 1, 95, 96, 4), (0, 1, 0, 2, 97, 98, 2)]:
        depth = dh + ds + dp
        n = 64 << depth
        ah = ref.random(1, n * n, sa)
        bh = ref.random(1, n * n, sb)
        c, cnt = ref.coordinate(ah, bh, dh, ds, dp, workers, scheme, counts=True)
        C["coordinate"].append({"d_host": dh, "d_serial": ds, "d_parallel": dp, "a_seed": sa, "b_seed": sb,
                                "scheme": scheme, "workers": workers, "counts": [int(x) for x in cnt], **digest(c)})

    C["predicted_additions"] = []
    for scheme in (0, 1, 2):
        for depth in (1, 2, 3, 4):
            C["predicted_additions"].append({"scheme": scheme, "depth": depth,
                                             "basis": ref.predicted_additions(scheme, depth, 0),
                                             "lin": ref.predicted_additions(scheme, depth, 1)})
    OUT.write_text(json.dumps(g, indent=1))
    print("wrote", OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
