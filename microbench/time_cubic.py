"""Quick device-resident timing of the panel product kernels (dev helper, not the bench)."""
from __future__ import annotations

import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402


def run(n: int, kernel: int, ring: int, reps: int = 5) -> dict:
    lib = bmm.lib()
    gm, gn, gk = bmm.granularity(kernel)
    kw = n // 64
    dA = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
    dBt = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
    dC = torch.empty((n, n // 64), dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    for _ in range(2):
        assert lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dBt.data_ptr(), kw, dC.data_ptr(), n // 64, n, n, kw, ring,
                                    kernel, 0, sp) == 0, lib.bmmgpu_last_error()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dBt.data_ptr(), kw, dC.data_ptr(), n // 64, n, n, kw, ring, kernel, 0,
                             sp)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    bops = 2.0 * n**3 - n * n
    return {"n": n, "kernel": kernel, "ring": ring, "ms": ms, "eff_Pbops": bops / (ms * 1e-3) / 1e15}


if __name__ == "__main__":
    kernels = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1"])]
    sizes = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["8192", "16384"])]
    for k in kernels:
        for n in sizes:
            for ring in (1, 0):
                print(json.dumps(run(n, k, ring)), flush=True)
