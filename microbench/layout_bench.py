"""Throughput of the layout conversions (csrc/layout.cu, the reference
CLI's `transform`, tools/bmm_cli.cpp:210-234):

  device: bmmgpu_dev_layout on an n x n matrix in HBM, CUDA events; algorithmic bytes
          = 2 n^2 / 8 (read once, write once) against the HBM copy peak;
  host:   bmmgpu_layout from / to page-locked host buffers, streamed through the GPU in
          super-tiles; bytes over the link = 2 n^2 / 8 (up and down).

    python microbench/layout_bench.py [n_device] [n_host]
"""
from __future__ import annotations

import ctypes
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

OPS = {"transpose_blocks64": bmm.LAYOUT_TRANSPOSE_BLOCKS64, "to_interleaved_right": bmm.LAYOUT_TO_INTERLEAVED_RIGHT,
       "from_interleaved": bmm.LAYOUT_FROM_INTERLEAVED}


def device(n: int, reps: int = 5) -> None:
    L = bmm.lib()
    words = n * n // 64
    src = torch.randint(-2**62, 2**62, (words,), dtype=torch.int64, device="cuda")
    dst = torch.empty_like(src)
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for name, op in OPS.items():
        out = src if op == bmm.LAYOUT_TRANSPOSE_BLOCKS64 else dst
        assert L.bmmgpu_dev_layout(src.data_ptr(), out.data_ptr(), n, n, op, sp) == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            assert L.bmmgpu_dev_layout(src.data_ptr(), out.data_ptr(), n, n, op, sp) == 0
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = 2 * words * 8 / (ms * 1e-3) / 1e9
        print(json.dumps({"where": "device", "op": name, "n": n, "ms": round(ms, 3), "GB_per_s": round(gbs, 1)}),
              flush=True)


def host(n: int, reps: int = 2) -> None:
    words = n * n // 64
    a = bmm.PinnedWords(words)
    b = bmm.PinnedWords(words)
    try:
        a.words[:] = np.arange(words, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        for name, op in OPS.items():
            dst = a.words if op == bmm.LAYOUT_TRANSPOSE_BLOCKS64 else b.words
            bmm.layout(a.words, dst, n, n, op)
            t0 = time.perf_counter()
            for _ in range(reps):
                bmm.layout(a.words, dst, n, n, op)
            s = (time.perf_counter() - t0) / reps
            print(json.dumps({"where": "host-streamed (pinned)", "op": name, "n": n, "s": round(s, 3),
                              "GB_per_s_each_way": round(words * 8 / s / 1e9, 1),
                              "per_Tib_s": round(s * (2**40 / (n * n)), 2)}), flush=True)
        # pageable source / destination (numpy memory): staged copies
        pa = np.empty(words, dtype=np.uint64)
        pa[:] = a.words
        pb = np.empty_like(pa)
        t0 = time.perf_counter()
        bmm.layout(pa, pb, n, n, bmm.LAYOUT_TO_INTERLEAVED)
        s = time.perf_counter() - t0
        print(json.dumps({"where": "host-streamed (pageable)", "op": "to_interleaved", "n": n, "s": round(s, 3),
                          "GB_per_s_each_way": round(words * 8 / s / 1e9, 1)}), flush=True)
    finally:
        a.free()
        b.free()


if __name__ == "__main__":
    nd = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    nh = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
    device(nd)
    host(nh)
