"""First-call cost of the public fast path in a fresh process: wall time
of three consecutive bmm.multiply calls (alt-si, n = 65536 by default) from page-locked
buffers, plus the time of the first CUDA context / library setup on its own.

    python microbench/first_call.py [n] [init: none | plain | reserve]

init: none = no warm-up; plain = bmm.init() (kernels and stream pool); reserve = bmm.init()
with 16 GiB reserved in the memory pool.  The warm-up is timed on its own.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

t_start = time.perf_counter()
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402


def main() -> None:
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    mode = sys.argv[2] if len(sys.argv) > 2 else "none"
    t0 = time.perf_counter()
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    t_ctx = time.perf_counter() - t0
    t1 = time.perf_counter()
    if mode != "none":
        bmm.init(0, (16 << 30) if mode == "reserve" else 0)
    t_init = time.perf_counter() - t1
    w = n * n // 64
    a, b, c = bmm.PinnedWords(w), bmm.PinnedWords(w), bmm.PinnedWords(w)
    bmm.random_rows_into(a.words, n, 1, 0, n)
    bmm.random_rows_into(b.words, n, 2, 0, n)
    plan = bmm.LayerPlan.auto_plan(n, 1)
    times = []
    for _ in range(4):
        s = time.perf_counter()
        bmm.multiply(bmm.BitMatrix(n, n, a.words), bmm.BitMatrix(n, n, b.words), bmm.Algo.AltSelfInverse, plan,
                     bmm.Semiring.Gf2XorAnd, out=bmm.BitMatrix(n, n, c.words))
        times.append(time.perf_counter() - s)
    eff = 2.0 * n**3 - n * n
    print(json.dumps({"n": n, "init": mode, "init_s": round(t_init, 3), "import_s": round(t0 - t_start, 3),
                      "context_s": round(t_ctx, 3),
                      "call_s": [round(t, 4) for t in times], "first_over_warm": round(times[0] / min(times[1:]), 2),
                      "Pbops_per_call": [round(eff / t / 1e15, 2) for t in times]}), flush=True)


if __name__ == "__main__":
    main()
