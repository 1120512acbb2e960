"""Where the persistent tcgen05 kernel loses time on a batch of short-K leaf products
(dev helper; needs a -DBMMGPU_PROBE build, tools/build_variant.py probe cubic_umma2.cu -DBMMGPU_PROBE).

    BMMGPU_UMMA_PROBE=<v> python microbench/probe_leaf.py [L] [batch]

Prints the launch time and, averaged over CTAs, the fraction of each role's loop time
spent in each barrier wait (probe v = 0: the real kernel with wait accounting).
"""
from __future__ import annotations

import ctypes
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1200
lib = bmm.lib()
kw = L // 64
dA = torch.randint(-2**62, 2**62, (batch, L, kw), dtype=torch.int64, device="cuda")
dBt = torch.randint(-2**62, 2**62, (batch, L, kw), dtype=torch.int64, device="cuda")
dC = torch.empty((batch, L, L // 64), dtype=torch.int64, device="cuda")
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def go():
    st = lib.bmmgpu_dev_cubic_batched(dA.data_ptr(), kw, L * kw, dBt.data_ptr(), kw, L * kw, dC.data_ptr(),
                                      L // 64, L * (L // 64), batch, L, L, kw, 1, 2, 0, sp)
    assert st == 0, lib.bmmgpu_last_error()


for _ in range(2):
    go()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    go()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
out = {"probe": os.environ.get("BMMGPU_UMMA_PROBE", ""), "L": L, "batch": batch, "ms": round(ms, 3),
       "Pbops": round(batch * (2.0 * L**3 - L * L) / (ms * 1e-3) / 1e15, 3),
       "us_per_tile": round(ms * 1e3 / (batch * (L // 256) ** 2 / 74), 3)}
buf = (ctypes.c_ulonglong * (148 * 8))()
if lib.bmmgpu_debug_umma2_probe(buf) == 0:
    rows = [[buf[c * 8 + i] for i in range(8)] for c in range(148)]

    def frac(idx, tot, ctas):
        v = [rows[c][idx] / rows[c][tot] for c in ctas if rows[c][tot]]
        return round(sum(v) / max(1, len(v)), 4)

    leaders = range(0, 148, 2)
    out.update({"expander_wait_empty": frac(0, 2, range(148)), "expander_wait_packed": frac(1, 2, range(148)),
                "mma_wait_full": frac(3, 5, leaders), "mma_wait_acc": frac(4, 5, leaders),
                "loader_wait_packed_empty": frac(6, 7, range(148)),
                # effective SM clock: the MMA lane's loop cycles (clock64) over the last launch's time
                "eff_mhz": round(sum(rows[c][5] for c in leaders) / len(leaders) / (ms * 1e3), 1)})
print(json.dumps(out), flush=True)
