"""Pinned host <-> device bandwidth of 2-D copies by row width (dev helper): the
streamed drivers move quadrants / sub-blocks of row-major bit matrices, i.e. copies
whose rows are n/128 or n/256 words of a longer host row."""
import json
import sys
import time

import torch
from cuda.bindings import runtime as rt

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = n // 64
h = torch.empty(n * w, dtype=torch.int64, pin_memory=True)
d = torch.empty(n * w, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for kind_name, kind in (("h2d", rt.cudaMemcpyKind.cudaMemcpyHostToDevice),
                        ("d2h", rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)):
    for parts in (1, 2, 4, 8):  # row width = w / parts words, n / parts rows... one block of (n/parts)^2 bits
        width = (w // parts) * 8
        rows = n // parts
        nbytes = width * rows
        src, dst = (h.data_ptr(), d.data_ptr()) if kind_name == "h2d" else (d.data_ptr(), h.data_ptr())
        for it in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = 4
            for _ in range(reps):
                (err,) = rt.cudaMemcpy2DAsync(dst, w * 8, src, w * 8, width, rows, kind, s)
                assert err == rt.cudaError_t.cudaSuccess, err
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / reps
        print(json.dumps({"dir": kind_name, "row_bytes": width, "rows": rows, "MiB": nbytes / 2**20,
                          "GBps": nbytes / dt / 1e9}), flush=True)
