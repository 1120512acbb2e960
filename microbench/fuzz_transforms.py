"""Randomised differential test of the layout, basis-change and alt-basis product entry points
against the unmodified reference (oracle/_ref) -- dev helper, GPU box:
  bmmgpu_layout: transpose_blocks64 on random block shapes, to / from_interleaved (left, right)
    at random depths;
  bmmgpu_basis_change: phi / psi / chi of every scheme at random depths, in core and streamed
    beyond a small forced budget (BMMGPU_BASIS_BUDGET);
  bmmgpu_multiply_alt: every scheme at random depths.

    python microbench/fuzz_transforms.py [seconds] [seed]
"""
from __future__ import annotations

import ctypes
import json
import os
import random
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402
from oracle import Reference  # noqa: E402

budget_s = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = random.Random(seed)
ref = Reference()
lib = bmm.lib()
P = lambda a: a.ctypes.data  # noqa: E731
BUILTIN = {1: 0, 2: 1, 3: 2}  # bmmgpu algo id -> bmm::Builtin (StrassenWinograd, AltSelfInverse, AltChaining)


def case_layout(i: int):
    kind = rng.choice(["transpose", "to", "from"])
    if kind == "transpose":
        rows, cols = 64 * rng.randint(1, 64), 64 * rng.randint(1, 64)
        m = ref.random(rows, cols, 100 + i)
        want = ref.transpose_blocks64(rows, cols, m)
        got = np.empty_like(m)
        st = lib.bmmgpu_layout(P(m), P(got), rows, cols, 0, None)
        return {"op": "transpose_blocks64", "rows": rows, "cols": cols}, st, got, want
    depth = rng.randint(0, 7)
    n = 64 << depth
    which = rng.choice([0, 1])  # bmm::Operand Left / Right
    m = ref.random(n, n, 200 + i)
    if kind == "to":
        want = ref.to_interleaved(depth, which, m)
        got = np.empty_like(m)
        st = lib.bmmgpu_layout(P(m), P(got), n, n, 2 if which else 1, None)
    else:
        want = ref.from_interleaved(depth, which, m)
        got = np.empty_like(m)
        st = lib.bmmgpu_layout(P(m), P(got), n, n, 4 if which else 3, None)
    return {"op": kind + "_interleaved", "depth": depth, "which": which}, st, got, want


def case_basis(i: int):
    depth = rng.randint(1, 7)
    algo = rng.choice([2, 3, 1])
    factor = rng.choice([0, 1, 2])
    n = 64 << depth
    v = ref.random(n, n, 300 + i)
    want = ref.basis_change(v, depth, factor, BUILTIN[algo])
    got = v.copy()
    streamed = rng.random() < 0.4
    if streamed:
        os.environ["BMMGPU_BASIS_BUDGET"] = str(max(64 * 1024, (v.nbytes // rng.choice([2, 4, 8]))))
    st = lib.bmmgpu_basis_change(P(got), got.size, depth, algo, factor, 0)
    os.environ.pop("BMMGPU_BASIS_BUDGET", None)
    return {"op": "basis_change", "depth": depth, "algo": algo, "factor": factor, "streamed": streamed}, st, got, want


def case_alt(i: int):
    depth = rng.randint(1, 5)
    algo = rng.choice([2, 3, 1])
    n = 64 << depth
    a = ref.random(n, n, 400 + i)
    b = ref.random(n, n, 500 + i)
    ds = rng.randint(0, depth)
    want = ref.multiply_alt(a, b, ds, depth - ds, 1, BUILTIN[algo])
    got = np.zeros_like(a)
    st = lib.bmmgpu_multiply_alt(P(a), P(b), P(got), depth, algo, None)
    return {"op": "multiply_alt", "depth": depth, "algo": algo}, st, got, want


t0 = time.time()
done = fails = 0
i = 0
while time.time() - t0 < budget_s:
    i += 1
    case, st, got, want = rng.choice([case_layout, case_layout, case_basis, case_alt])(i)
    done += 1
    if st != 0:
        fails += 1
        print(json.dumps({**case, "status": st, "error": lib.bmmgpu_last_error().decode()}), flush=True)
    elif not np.array_equal(got, want):
        fails += 1
        print(json.dumps({**case, "mismatched_words": int(np.count_nonzero(got != want))}), flush=True)
print(json.dumps({"cases": done, "failures": fails, "seconds": round(time.time() - t0, 1), "seed": seed}), flush=True)
sys.exit(1 if fails else 0)
