"""Host-API products from pageable vs page-locked buffers (dev helper): median wall
time of bmmgpu_multiply (alt-si) and bmmgpu_cubic at n, buffers pre-touched."""
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = n // 64
lib = bmm.lib()
a = np.empty(n * w, dtype=np.uint64)
b = np.empty(n * w, dtype=np.uint64)
bmm.random_rows_into(a, n, 1, 0, n)
bmm.random_rows_into(b, n, 2, 0, n)
c = np.ones(n * w, dtype=np.uint64)
pa = torch.from_numpy(a.view(np.int64)).pin_memory()
pb = torch.from_numpy(b.view(np.int64)).pin_memory()
pc = torch.zeros(n * w, dtype=torch.int64).pin_memory()
plan = bmm._Plan(0, 0, (n // 64).bit_length() - 1, 1, 1)
for label, (A, B, C) in (("pageable", (a.ctypes.data, b.ctypes.data, c.ctypes.data)),
                         ("pinned", (pa.data_ptr(), pb.data_ptr(), pc.data_ptr()))):
    for name, call in (("alt-si", lambda: lib.bmmgpu_multiply(A, B, C, n, 2, ctypes.byref(plan), 1, None)),
                       ("cubic", lambda: lib.bmmgpu_cubic(A, B, C, n, n, n, 1, None))):
        call()
        ts = []
        for _ in range(3):
            s0 = time.perf_counter()
            assert call() == 0, lib.bmmgpu_last_error()
            ts.append(time.perf_counter() - s0)
        t = statistics.median(ts)
        print(json.dumps({"buffers": label, "call": name, "staging": os.environ.get("BMMGPU_NO_STAGING") is None,
                          "s": t, "Pbops": (2.0 * n**3 - n * n) / t / 1e15}), flush=True)
