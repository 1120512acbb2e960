"""A/B of the host-buffer fast path between two builds of libbmmgpu.so (only the stable
ABI: bmmgpu_multiply from page-locked buffers), several calls each, alternating builds.

    python microbench/e2e_host_ab.py LIB_A LIB_B [n] [rounds]
"""
from __future__ import annotations

import ctypes
import json
import subprocess
import sys
import time

CHILD = r"""
import ctypes, json, sys, time, torch
lib = ctypes.CDLL(sys.argv[1])
n = int(sys.argv[2])
class Opts(ctypes.Structure):
    _fields_ = [("device_mask", ctypes.c_uint32), ("kernel", ctypes.c_int32), ("accumulate", ctypes.c_int32),
                ("leaf_log2", ctypes.c_int32), ("timing_ms", ctypes.POINTER(ctypes.c_double)),
                ("device_budget", ctypes.c_uint64), ("force_streaming", ctypes.c_int32), ("reserved", ctypes.c_int32)]
class Plan(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in ("d_host", "d_serial", "d_parallel", "d_inner", "workers")]
w = n * n // 64
g = torch.Generator().manual_seed(1)
a = torch.randint(-2**62, 2**62, (w,), dtype=torch.int64, generator=g).pin_memory()
b = torch.randint(-2**62, 2**62, (w,), dtype=torch.int64, generator=g).pin_memory()
c = torch.empty(w, dtype=torch.int64).pin_memory()
depth = (n // 64).bit_length() - 1
p = Plan(0, depth - min(3, depth), min(3, depth), 1, 1)
lib.bmmgpu_multiply.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint64, ctypes.c_int32, ctypes.POINTER(Plan),
                                ctypes.c_int32, ctypes.POINTER(Opts)]
o = Opts()
ts = []
for _ in range(8):
    s = time.perf_counter()
    assert lib.bmmgpu_multiply(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, 2, ctypes.byref(p), 1, ctypes.byref(o)) == 0
    ts.append(time.perf_counter() - s)
print(json.dumps([round(t * 1e3, 2) for t in ts]))
"""


def main() -> None:
    libs = sys.argv[1:3]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    for r in range(rounds):
        for lib in libs:
            out = subprocess.run([sys.executable, "-c", CHILD, lib, str(n)], capture_output=True, text=True)
            print(json.dumps({"round": r, "lib": lib, "ms": json.loads(out.stdout.strip().splitlines()[-1])
                              if out.returncode == 0 else out.stderr[-500:]}), flush=True)


if __name__ == "__main__":
    main()
