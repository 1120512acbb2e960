"""Standalone basis change (bmm_cli `transform`) of an interleaved vector larger than
the device budget (dev helper): n = 2^19 operand (32 GiB) with a 12 GiB budget,
pinned host buffer.  Prints seconds and effective host<->device GB/s."""
import ctypes
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 13   # n = 64 * 2^13 = 2^19
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 12 << 30
words = (4 ** depth) * 64
h = torch.empty(words, dtype=torch.int64, pin_memory=True)
hn = h.numpy().view(np.uint64)
hn[:] = np.arange(words, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
lib = bmm.lib()
os.environ["BMMGPU_BASIS_BUDGET"] = str(budget)
for inverse in (0, 1):
    t0 = time.perf_counter()
    assert lib.bmmgpu_basis_change(h.data_ptr(), words, depth, 2, 0, inverse) == 0, lib.bmmgpu_last_error()
    t = time.perf_counter() - t0
    h2d, d2h = ctypes.c_uint64(0), ctypes.c_uint64(0)
    print(json.dumps({"depth": depth, "GiB": words * 8 / 2**30, "budget_GiB": budget / 2**30, "inverse": inverse,
                      "s": t, "link_GBps": (words * 8 * 2 * (1 + 2)) / t / 1e9}), flush=True)
ok = np.array_equal(hn[:1 << 20], np.arange(1 << 20, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15))
print(json.dumps({"roundtrip_ok_first_8MiB": bool(ok)}))
