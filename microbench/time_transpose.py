"""Device time of K3 (bmmgpu_dev_transpose, B -> Bt) at n x n (dev helper): GB/s of algorithmic
traffic (n^2/8 bytes read + the same written)."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

lib = bmm.lib()
for n in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["65536", "131072"])]:
    w = n // 64
    dB = torch.randint(-2**62, 2**62, (n, w), dtype=torch.int64, device="cuda")
    dBt = torch.empty((n, w), dtype=torch.int64, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        assert lib.bmmgpu_dev_transpose(dB.data_ptr(), w, n, n, dBt.data_ptr(), n, w, sp) == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        lib.bmmgpu_dev_transpose(dB.data_ptr(), w, n, n, dBt.data_ptr(), n, w, sp)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"n": n, "ms": round(ms, 4), "GBps": round(2 * n * n / 8 / (ms * 1e-3) / 1e9, 1)}), flush=True)
