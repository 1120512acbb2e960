"""Where the end-to-end time of bmmgpu_cubic goes (dev helper): pinned H2D / D2H
bandwidth, wall time of the call against its device-side span (timing_ms), and
the library's copy byte counts."""
import ctypes
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 131072
w = n // 64
lib = bmm.lib()
h = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
d = torch.empty(n * w, dtype=torch.int64, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(json.dumps({name + "_GBps": n * w * 8 / dt / 1e9}))
del d
hA = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
hC = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
bmm.random_rows_into(hA.numpy().view(np.uint64), n, 1, 0, n)
bmm.random_rows_into(h.numpy().view(np.uint64), n, 2, 0, n)
import os
# each case: "-" (defaults) or "VAR=val,VAR=val" library knobs; argv[2:] or the slice A/B
case_args = [a for a in sys.argv[1:] if not a.isdigit() and a != "--all"]
if not case_args:
    case_args = ["BMMGPU_KOUTER_SLICES=equal", "-", "BMMGPU_KOUTER_SLICES=3,64", "BMMGPU_KOUTER_SLICES=2,32"]
knobs = sorted({kv.split("=")[0] for c in case_args if c != "-" for kv in c.split(",")})
cases = [(0, None, c) for _ in range(3) for c in case_args]
if "--all" in sys.argv:
    cases += [(1, None, "-"), (2, "2", "-"), (2, "3", "-"), (2, "4", "-"), (2, "8", "-")]
for mode, chunks, case in cases:
    for kname in knobs + ["BMMGPU_KOUTER_CHUNKS"]:
        os.environ.pop(kname, None)
    if case != "-":
        for kv in case.split(","):
            kk, vv = kv.split("=", 1)
            os.environ[kk] = vv
    if chunks:
        os.environ["BMMGPU_KOUTER_CHUNKS"] = chunks
    slices = case
    t = ctypes.c_double(0)
    opts = bmm._opts(0, timing=t, device_mask=1, force_streaming=mode)
    walls = []
    for rep in range(int(os.environ.get('DIAG_REPS', '4'))):
        lib.bmmgpu_block_timer(1)
        s0 = time.perf_counter()
        assert lib.bmmgpu_cubic(hA.data_ptr(), h.data_ptr(), hC.data_ptr(), n, n, n, 0, ctypes.byref(opts)) == 0
        wall = time.perf_counter() - s0
        walls.append(wall)
        bms, bl = ctypes.c_double(0), ctypes.c_uint64(0)
        lib.bmmgpu_block_timer_read(ctypes.byref(bms), ctypes.byref(bl))
        lib.bmmgpu_block_timer(0)
    h2d, d2h = ctypes.c_uint64(0), ctypes.c_uint64(0)
    lib.bmmgpu_last_copy_bytes(ctypes.byref(h2d), ctypes.byref(d2h))
    print(json.dumps({"force_streaming": mode, "chunks": chunks, "slices": slices, "wall_ms": wall * 1e3, "walls_ms": [round(x * 1e3, 1) for x in walls], "device_span_ms": t.value,
                      "block_ms": bms.value, "block_launches": bl.value,
                      "h2d_GB": h2d.value / 1e9, "d2h_GB": d2h.value / 1e9,
                      "Pbops": (2.0 * n**3 - n * n) / wall / 1e15}), flush=True)
