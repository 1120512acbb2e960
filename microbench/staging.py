"""Staged (pageable) vs direct (page-locked) host copies through the C ABI, isolated:
bmmgpu_cubic with a tiny inner or outer dimension so one operand's copy dominates (dev helper).
  upload:   m = 256, k = n = N  -> B (N^2/8 bytes) goes up, C and A are small
  download: m = N, k = 64, n = N -> C (N^2/8 bytes) comes down, A and B are small"""
import ctypes
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
lib = bmm.lib()
for what, (m, k, n) in (("upload", (256, N, N)), ("download", (N, 64, N))):
    sizes = (m * ((k + 63) // 64), k * ((n + 63) // 64), m * ((n + 63) // 64))
    for kind in ("pageable", "pinned"):
        bufs = []
        for sz in sizes:
            x = np.ones(sz, dtype=np.uint64)
            bufs.append(torch.from_numpy(x.view(np.int64)).pin_memory() if kind == "pinned" else x)
        ptr = [b.data_ptr() if kind == "pinned" else b.ctypes.data for b in bufs]
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            assert lib.bmmgpu_cubic(ptr[0], ptr[1], ptr[2], m, k, n, 1, None) == 0, lib.bmmgpu_last_error()
            ts.append(time.perf_counter() - t0)
        t = statistics.median(ts[1:])
        moved = (sizes[1] if what == "upload" else sizes[2]) * 8
        print(json.dumps({"copy": what, "buffers": kind, "bytes": moved, "s": round(t, 4),
                          "GBps": round(moved / t / 1e9, 1)}), flush=True)
