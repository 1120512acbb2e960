"""Device-resident timing of a batch of L x L x L products in one persistent launch
(the leaf layer of the fast recursion) -- dev helper, not the bench.

    python microbench/time_leaf.py [L list] [batch list]
"""
from __future__ import annotations

import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402


def run(L: int, batch: int, ring: int = 1, kernel: int = 2, reps: int = 3) -> dict:
    lib = bmm.lib()
    kw = L // 64
    dA = torch.randint(-2**62, 2**62, (batch, L, kw), dtype=torch.int64, device="cuda")
    dBt = torch.randint(-2**62, 2**62, (batch, L, kw), dtype=torch.int64, device="cuda")
    dC = torch.empty((batch, L, L // 64), dtype=torch.int64, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def go():
        st = lib.bmmgpu_dev_cubic_batched(dA.data_ptr(), kw, L * kw, dBt.data_ptr(), kw, L * kw, dC.data_ptr(),
                                          L // 64, L * (L // 64), batch, L, L, kw, ring, kernel, 0, sp)
        assert st == 0, lib.bmmgpu_last_error()

    go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        go()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    bops = batch * (2.0 * L**3 - L * L)
    tiles = batch * (L // 256) ** 2
    return {"L": L, "batch": batch, "ms": ms, "Pbops": bops / (ms * 1e-3) / 1e15,
            "us_per_tile_per_pair": ms * 1e3 / (tiles / 74)}


if __name__ == "__main__":
    Ls = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2048", "4096", "8192"])]
    for L in Ls:
        batch = {2048: 16807 // 4, 4096: 2401 // 2, 8192: 343 // 2}.get(L, 64)
        print(json.dumps(run(L, batch)), flush=True)
