"""Where the persistent tcgen05 kernel's roles wait (dev helper; needs a
-DBMMGPU_PROBE build of libbmmgpu.so, see microbench/variant_lib.sh).

    BMMGPU_UMMA_PROBE=<v> python microbench/probe_waits.py <n>

Prints, averaged over CTAs, the fraction of each role's loop time spent in each
barrier wait: expander warp 0 (empty / packed-full), MMA lane (full / acc_empty,
leader CTAs), loader warp 0 (packed-empty).
"""
from __future__ import annotations

import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
lib = bmm.lib()
kw = n // 64
dA = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
dBt = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
dC = torch.empty((n, n // 64), dtype=torch.int64, device="cuda")
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    assert lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dBt.data_ptr(), kw, dC.data_ptr(), n // 64, n, n, kw, 1, 2, 0, sp) == 0
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (148 * 8))()
assert lib.bmmgpu_debug_umma2_probe(buf) == 0, "not a -DBMMGPU_PROBE build"
rows = [[buf[c * 8 + i] for i in range(8)] for c in range(148)]


def frac(idx: int, tot: int, ctas) -> float:
    v = [rows[c][idx] / rows[c][tot] for c in ctas if rows[c][tot]]
    return sum(v) / max(1, len(v))


leaders = range(0, 148, 2)
print(json.dumps({
    "n": n,
    "expander_wait_empty": frac(0, 2, range(148)),
    "expander_wait_packed": frac(1, 2, range(148)),
    "mma_wait_full": frac(3, 5, leaders),
    "mma_wait_acc_empty": frac(4, 5, leaders),
    "loader_wait_packed_empty": frac(6, 7, range(148)),
    "loop_cycles_mma": sum(rows[c][5] for c in leaders) / len(leaders),
}))
