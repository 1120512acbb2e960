"""Copy floor of a small end-to-end product (dev helper, GPU box): pinned H2D of A + B and
D2H of C for n = 8192 alone (sequential and with the download on a second stream), against
bmmgpu_cubic's wall time at the same n."""
import json
import statistics
import time

import torch

n = 8192
w = n // 64
hA = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
hB = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
hC = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
dA = torch.empty(n * w, dtype=torch.int64, device="cuda")
dB = torch.empty(n * w, dtype=torch.int64, device="cuda")
dC = torch.empty(n * w, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(f, reps=50):
    walls = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    return statistics.median(walls[5:]) * 1e6


def h2d():
    with torch.cuda.stream(s1):
        dA.copy_(hA, non_blocking=True)
        dB.copy_(hB, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        hC.copy_(dC, non_blocking=True)


def both():
    h2d()
    d2h()


for name, f in (("h2d_16MiB", h2d), ("d2h_8MiB", d2h), ("h2d_and_d2h_concurrent", both)):
    us = timed(f)
    print(json.dumps({"op": name, "us": round(us, 1)}))
