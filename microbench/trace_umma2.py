"""Pipeline timestamps of the persistent tcgen05 kernel, pair 0, stages 0..511
(needs a -DBMMGPU_TRACE build; BMMGPU_UMMA_TRACE=1 is set here).  Global timer, ns."""
import ctypes, os, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["BMMGPU_UMMA_TRACE"] = "1"
import paper_1909_01554_b200 as bmm
lib = bmm.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4
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
e0, e1, r0, r1 = a[1024:1536], a[2048:2560], a[1536:2048], a[2560:3072]
t0 = full[0]
print("it   full  commit  empty0 empty1 arrive0 arrive1  (ns from full[0])")
for it in range(0, 80):
    print(f"{it:3d} {full[it]-t0:6d} {commit[it]-t0:6d} {e0[it]-t0:6d} {e1[it]-t0:6d} {r0[it]-t0:6d} {r1[it]-t0:6d}")
rows = []
for it in range(S + 8, 500):
    rows.append([e0[it] - commit[it - S], r0[it] - e0[it], r1[it] - e1[it], full[it] - max(r0[it], r1[it]),
                 full[it] - full[it - 1], commit[it] - full[it]])
r = np.array(rows)
names = ["commit(it-S) issued -> empty seen CTA0", "empty -> arrive CTA0", "empty -> arrive CTA1",
         "last arrive -> full seen", "full(it) - full(it-1)", "full -> commit issued"]
for k, col in zip(names, r.T):
    print(f"{k:40s} median {np.median(col):7.0f}  p90 {np.percentile(col, 90):7.0f} ns")
