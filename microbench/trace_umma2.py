"""Pipeline timestamps of the persistent tcgen05 kernel (debug flag 16)."""
import ctypes, os, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
os.environ["BMMGPU_UMMA_DEBUG"] = str(16 | mode)
lib = bmm.lib()
n = 16384; kw = n // 64
dA = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
dB = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
dC = torch.empty((n, n // 64), dtype=torch.int64, device="cuda")
for _ in range(2):
    assert lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dB.data_ptr(), kw, dC.data_ptr(), n // 64, n, n, kw, 1, 2, 0, None) == 0
torch.cuda.synchronize()
t = (ctypes.c_ulonglong * 2560)()
lib.bmmgpu_debug_umma2_trace(t)
a = np.array(t, dtype=np.int64)
full, commit, empty, arr0, arr7 = a[:512], a[512:1024], a[1024:1536], a[1536:2048], a[2048:2560]
base = full[0]
S = 6
print("mode", mode)
for it in list(range(0, 24)) + list(range(200, 212)):
    line = f"it {it:3d} full {full[it]-base:8d} commit {commit[it]-base:8d}"
    if it >= S:
        line += f" | empty(it) {empty[it]-base:8d} arr0 {arr0[it]-base:8d} arr7 {arr7[it]-base:8d}"
        line += f" | commit(it-6)->empty {empty[it]-commit[it-S]:6d} arrive->full {full[it]-max(arr0[it],arr7[it]):6d}"
    print(line)
d = np.diff(full[50:500])
print("cycles per stage (median, mean):", np.median(d), d.mean())
