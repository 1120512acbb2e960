"""Host enqueue time vs device time of bmmgpu_dev_multiply (dev helper)."""
from __future__ import annotations

import ctypes
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 12
lib = bmm.lib()
w = n // 64
dA0 = torch.randint(-2**62, 2**62, (n, w), dtype=torch.int64, device="cuda")
dB = torch.randint(-2**62, 2**62, (n, w), dtype=torch.int64, device="cuda")
dA = torch.empty_like(dA0)
dBt = torch.empty(((n + 255) // 256 * 256, w), dtype=torch.int64, device="cuda")
dC = torch.empty((n, w), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
sp = ctypes.c_void_p(s.cuda_stream)
for rep in range(4):
    dA.copy_(dA0)
    dBt[:n].copy_(dB)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    rc = lib.bmmgpu_dev_multiply(dA.data_ptr(), w, dBt.data_ptr(), w, dC.data_ptr(), w, n, 2, leaf, 0, sp)
    e1.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    h2 = time.perf_counter()
    print(f"rep {rep} rc {rc} enqueue {1e3 * (h1 - h0):.1f} ms  total {1e3 * (h2 - h0):.1f} ms  "
          f"device {e0.elapsed_time(e1):.1f} ms", flush=True)
