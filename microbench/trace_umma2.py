"""Cross-CTA pipeline timestamps of the persistent tcgen05 kernel (BMMGPU_UMMA_TRACE=1)."""
import ctypes, os, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["BMMGPU_UMMA_TRACE"] = "1"
import paper_1909_01554_b200 as bmm
lib = bmm.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
kw = n // 64
dA = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
dB = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
dC = torch.empty((n, n // 64), dtype=torch.int64, device="cuda")
for _ in range(2):
    assert lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dB.data_ptr(), kw, dC.data_ptr(), n // 64, n, n, kw, 1, 2, 0, None) == 0
torch.cuda.synchronize()
t = (ctypes.c_ulonglong * 6144)()
assert lib.bmmgpu_debug_umma2_trace(t) == 0
a = np.array(t, dtype=np.int64)
full, commit = a[0:512], a[512:1024]
e0, e1, r0, r1, r0w7, r1w7 = a[1024:1536], a[2048:2560], a[1536:2048], a[2560:3072], a[1536+3072:2048+3072], a[2560+3072:3072+3072]
S = 6
rows = []
for it in range(100, 500):
    rows.append([e0[it] - commit[it - S], e1[it] - commit[it - S], r0[it] - e0[it], r1[it] - e1[it],
                 full[it] - max(r0[it], r0w7[it]), full[it] - max(r1[it], r1w7[it]), commit[it] - full[it],
                 full[it] - full[it - 1]])
m = np.median(np.array(rows), axis=0)
names = ["commit(it-6)->empty CTA0", "commit(it-6)->empty CTA1", "empty->arrive CTA0 w0", "empty->arrive CTA1 w0",
         "last CTA0 arrive->full", "last CTA1 arrive->full", "full->commit (MMA issue)", "full(it)-full(it-1)"]
for k, v in zip(names, m):
    print(f"{k:28s} {v:8.0f} ns")
