"""Where the end-to-end time of the streamed fast path goes (dev helper): wall time of
bmmgpu_multiply from pinned buffers against its device span (timing) and the time
inside the block-product launches, for quadrant streaming (BMMGPU_ALT_STREAM_LEVELS=1)
and sub-block streaming (2: every child split into grandchildren, 3: first / last).
argv: n reps modes (comma list)."""
import ctypes
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = n // 64
lib = bmm.lib()
hA = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
hB = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
hC = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
bmm.random_rows_into(hA.numpy().view(np.uint64), n, 1, 0, n)
bmm.random_rows_into(hB.numpy().view(np.uint64), n, 2, 0, n)
A = bmm.BitMatrix(n, n, hA.numpy().view(np.uint64))
B = bmm.BitMatrix(n, n, hB.numpy().view(np.uint64))
plan = bmm.LayerPlan.auto_plan(n, 1)
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "2", "3"]
for levels in modes + modes:
    os.environ["BMMGPU_ALT_STREAM_LEVELS"] = levels
    walls, spans, blocks = [], [], []
    for rep in range(reps + 1):
        t = ctypes.c_double(0)
        lib.bmmgpu_block_timer(1)
        s0 = time.perf_counter()
        bmm.multiply(A, B, bmm.Algo.AltSelfInverse, plan, bmm.Semiring.Gf2XorAnd, timing=t,
                     out=bmm.BitMatrix(n, n, hC.numpy().view(np.uint64)))
        wall = time.perf_counter() - s0
        bms, bl = ctypes.c_double(0), ctypes.c_uint64(0)
        lib.bmmgpu_block_timer_read(ctypes.byref(bms), ctypes.byref(bl))
        lib.bmmgpu_block_timer(0)
        if rep:
            walls.append(wall * 1e3)
            spans.append(t.value)
            blocks.append(bms.value)
    print(json.dumps({"levels": levels, "n": n, "wall_ms": [round(x, 2) for x in walls],
                      "span_ms": [round(x, 2) for x in spans], "block_ms": [round(x, 2) for x in blocks],
                      "block_launches": bl.value,
                      "e2e_Pbops": (2.0 * n**3 - n * n) / (min(walls) / 1e3) / 1e15}), flush=True)
