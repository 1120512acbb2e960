"""Tile-boundary timestamps of the persistent tcgen05 kernel on a batch of leaf
products (pair 0; needs a -DBMMGPU_TRACE build).  Global timer, ns.

    python microbench/trace_tiles.py [L] [batch]
"""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["BMMGPU_UMMA_TRACE"] = "1"
import paper_1909_01554_b200 as bmm  # noqa: E402

lib = bmm.lib()
L = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
kw = L // 64
dA = torch.randint(-2**62, 2**62, (batch, L, kw), dtype=torch.int64, device="cuda")
dB = torch.randint(-2**62, 2**62, (batch, L, kw), dtype=torch.int64, device="cuda")
dC = torch.empty((batch, L, L // 64), dtype=torch.int64, device="cuda")
for _ in range(2):
    assert lib.bmmgpu_dev_cubic_batched(dA.data_ptr(), kw, L * kw, dB.data_ptr(), kw, L * kw, dC.data_ptr(), L // 64,
                                        L * L // 64, batch, L, L, kw, 1, 2, 0, None) == 0
torch.cuda.synchronize()
t = (ctypes.c_ulonglong * 6144)()
assert lib.bmmgpu_debug_umma2_trace(t) == 0
a = np.array(t, dtype=np.int64)
full = a[0:512]
tile = a[3072:3072 + 2048].reshape(512, 4)  # commit acc_full, epi seen, epi done, mma sees empty
S = L // 256  # stages per tile
t0 = full[0]
print(f"L={L}: {S} stages per tile; ns from the first full stage")
print("tile  last_commit  epi_seen  epi_done  mma_empty  next_full  | mma_tail  drain  handoff  full_after_empty  stage_period")
rows = []
for i in range(1, min(512 // S, 500) - 1):
    c, es, ed = tile[i][0], tile[i][1], tile[i][2]
    me = tile[i + 1][3]
    nf = full[S * (i + 1)] if S * (i + 1) < 512 else 0
    per = (full[S * i + S - 1] - full[S * i]) / max(S - 1, 1)
    rows.append([es - c, ed - es, me - ed, nf - me if nf else 0, per])
    if i < 12:
        print(f"{i:4d} {c - t0:10d} {es - t0:9d} {ed - t0:9d} {me - t0:9d} {nf - t0 if nf else 0:9d}  | "
              f"{es - c:7d} {ed - es:6d} {me - ed:7d} {nf - me if nf else 0:9d} {per:9.0f}")
r = np.array(rows)
for k, col in zip(["mma_tail (commit->epi sees full)", "drain", "handoff (done->mma sees empty)",
                   "first full after empty", "stage period"], r.T):
    print(f"{k:36s} median {np.median(col):8.0f} ns")
per_tile = [full[S * (i + 1)] - full[S * i] for i in range(1, 512 // S - 1)]
print(f"{'tile period (first stage to first stage)':36s} median {np.median(per_tile):8.0f} ns")
