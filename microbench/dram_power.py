"""Same tensor-core work with and without DRAM traffic (dev helper): the n x n x n
product (panels stream from HBM) against a batch of 512 x 512 x n products that all
read one broadcast pair of panels (everything L2-resident).  Prints ms and the
median SM clock of each, to size what the cubic kernel's DRAM re-reads cost under
the board power cap."""
import ctypes
import json
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
lib = bmm.lib()
kw = n // 64
dA = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
dB = torch.randint(-2**62, 2**62, (n, kw), dtype=torch.int64, device="cuda")
dC = torch.empty((n, n // 64), dtype=torch.int64, device="cuda")
P = 512
batch = (n // P) ** 2
dCb = torch.empty((batch, P, P // 64), dtype=torch.int64, device="cuda")


def full():
    assert lib.bmmgpu_dev_cubic(dA.data_ptr(), kw, dB.data_ptr(), kw, dC.data_ptr(), n // 64, n, n, kw, 1, 2, 0,
                                None) == 0


def bcast():
    assert lib.bmmgpu_dev_cubic_batched(dA.data_ptr(), kw, 0, dB.data_ptr(), kw, 0, dCb.data_ptr(), P // 64,
                                        P * P // 64, batch, P, P, kw, 1, 2, 0, None) == 0, lib.bmmgpu_last_error()


def clocks(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "200"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            out.append(line.strip())
    p.terminate()


for name, fn in (("full", full), ("broadcast", bcast), ("full", full), ("broadcast", bcast)):
    fn()
    torch.cuda.synchronize()
    stop, samples = threading.Event(), []
    th = threading.Thread(target=clocks, args=(stop, samples))
    th.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / 4
    sm = sorted(float(s.split(",")[0]) for s in samples if s)
    pw = sorted(float(s.split(",")[1]) for s in samples if s)
    print(json.dumps({"case": name, "ms": ms, "Pbops": (2.0 * n**3 - n * n) / ms / 1e12,
                      "sm_mhz": sm[len(sm) // 2] if sm else None, "power_w": pw[len(pw) // 2] if pw else None}),
          flush=True)
