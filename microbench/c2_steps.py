"""Per-step device time of the c2 device-resident step (transpose + bmmgpu_dev_multiply alt-si,
n = 65536) over many back-to-back steps, with the host enqueue time and the leaf launch's time
(block timer) per step: where the step-to-step spread of the c2 bench comes from (dev helper).

    python microbench/c2_steps.py [n] [steps]
"""
from __future__ import annotations

import ctypes
import json
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lib = bmm.lib()
w = n // 64
dA = torch.randint(-2**62, 2**62, (n, w), dtype=torch.int64, device="cuda")
dB = torch.randint(-2**62, 2**62, (n, w), dtype=torch.int64, device="cuda")
dBt = torch.empty((n, w), dtype=torch.int64, device="cuda")
dC = torch.empty((n, w), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
sp = ctypes.c_void_p(s.cuda_stream)


def step():
    assert lib.bmmgpu_dev_transpose(dB.data_ptr(), w, n, n, dBt.data_ptr(), n, w, sp) == 0
    assert lib.bmmgpu_dev_multiply(dA.data_ptr(), w, dBt.data_ptr(), w, dC.data_ptr(), w, n, 2, 12, 0, sp) == 0


for _ in range(3):
    step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
enq, blk = [], []
ev[0].record()
for i in range(steps):
    lib.bmmgpu_block_timer(1)
    h0 = time.perf_counter()
    step()
    enq.append((time.perf_counter() - h0) * 1e3)
    ev[i + 1].record()
torch.cuda.synchronize()
dev = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
print(json.dumps({"n": n, "device_ms": [round(x, 2) for x in dev], "enqueue_ms": [round(x, 2) for x in enq],
                  "median_ms": round(statistics.median(dev), 2), "max_ms": round(max(dev), 2),
                  "Pbops_median": round((2.0 * n**3 - n * n) / (statistics.median(dev) * 1e-3) / 1e15, 3)}))
# synchronous per-step: device time and the leaf kernel's time
rows = []
for i in range(8):
    lib.bmmgpu_block_timer(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    step()
    hq = (time.perf_counter() - h0) * 1e3
    e1.record()
    torch.cuda.synchronize()
    bms, bl = ctypes.c_double(0), ctypes.c_uint64(0)
    lib.bmmgpu_block_timer_read(ctypes.byref(bms), ctypes.byref(bl))
    rows.append((round(e0.elapsed_time(e1), 2), round(bms.value, 2), round(hq, 2)))
lib.bmmgpu_block_timer(0)
print(json.dumps({"sync_steps_device_leaf_enqueue_ms": rows}))
