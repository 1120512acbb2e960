"""Fixed cost of one bmmgpu_cubic call (dev helper): median wall time from pinned host
buffers for small n (n = 256 is almost all per-call overhead), per in-core slice count."""
import ctypes
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

lib = bmm.lib()
for n in (256, 1024, 4096, 8192):
    w = n // 64
    hA = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
    hB = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
    hC = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
    bmm.random_rows_into(hA.numpy().view(np.uint64), n, 1, 0, n)
    bmm.random_rows_into(hB.numpy().view(np.uint64), n, 2, 0, n)
    for sl in sys.argv[1:] or ["1", "4"]:
        os.environ["BMMGPU_INCORE_SLICES"] = sl
        t = ctypes.c_double(0)
        opts = bmm._opts(0, timing=t, device_mask=1)
        walls = []
        for rep in range(60):
            s0 = time.perf_counter()
            assert lib.bmmgpu_cubic(hA.data_ptr(), hB.data_ptr(), hC.data_ptr(), n, n, n, 1, ctypes.byref(opts)) == 0
            walls.append(time.perf_counter() - s0)
        walls = walls[10:]
        med = statistics.median(walls)
        print(json.dumps({"n": n, "slices": sl, "wall_us_median": round(med * 1e6, 1),
                          "wall_us_min": round(min(walls) * 1e6, 1), "device_ms": round(t.value, 4),
                          "Pbops": (2.0 * n**3 - n * n) / med / 1e15}), flush=True)
