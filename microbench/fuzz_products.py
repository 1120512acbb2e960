"""Randomised differential test of the host API against the oracle (dev helper, GPU box):
random shapes (odd sizes, K across the K-outer and kTs thresholds), both semirings, both
kernels, the in-core / out-of-core / K-outer drivers (force_streaming 0/1/2, small device
budgets), page-locked or pageable buffers, the accumulate flag; plus alt-si / alt-chain / sw
products at random powers of two and leaf sizes against the oracle's cubic product.

    python microbench/fuzz_products.py [seconds] [seed]

Prints one JSON line per case that fails and a summary line; exit status 1 on any failure.
"""
from __future__ import annotations

import ctypes
import json
import os
import random
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402
from oracle import Oracle  # noqa: E402

budget_s = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = random.Random(seed)
orc = Oracle()
lib = bmm.lib()


def host(words: np.ndarray, pinned: bool):
    if not pinned:
        return words, words.ctypes.data
    t = torch.from_numpy(words.view(np.int64)).pin_memory()
    return t, t.data_ptr()


def words_of(obj) -> np.ndarray:
    return obj.numpy().view(np.uint64) if isinstance(obj, torch.Tensor) else obj


def cubic_case(i: int) -> dict | None:
    shape_kind = rng.choice(["small", "odd", "longk", "tall", "wide"])
    if shape_kind == "small":
        m, k, n = rng.randint(1, 300), rng.randint(1, 700), rng.randint(1, 300)
    elif shape_kind == "odd":
        m, k, n = rng.randint(200, 2100), rng.randint(100, 5000), rng.randint(200, 2100)
    elif shape_kind == "longk":
        m, k, n = rng.choice([256, 512, 768, 1000]), rng.choice([32768, 33024, 40000, 65536, 70000]), \
            rng.choice([256, 512, 777])
    elif shape_kind == "tall":
        m, k, n = rng.randint(2000, 6000), rng.randint(64, 2000), rng.randint(64, 600)
    else:
        m, k, n = rng.randint(64, 600), rng.randint(64, 2000), rng.randint(2000, 6000)
    ring = rng.choice([0, 1])
    kernel = rng.choice([0, 0, 1])
    mode = rng.choice([0, 0, 1, 2])
    budget = 0 if mode == 0 else rng.choice([0, 8 << 20, 24 << 20, 64 << 20])
    pinned = rng.random() < 0.5
    accumulate = rng.random() < 0.25
    kw, nw = -(-k // 64), -(-n // 64)
    a = orc.random(m, k, 1000 + i)
    b = orc.random(k, n, 2000 + i)
    c0 = orc.random(m, n, 3000 + i) if accumulate else np.zeros(m * nw, dtype=np.uint64)
    want = orc.multiply_cubic(a, b, m, k, n, ring)
    if accumulate:
        want = (c0 ^ want) if ring == 1 else (c0 | want)
    ha, pa = host(a, pinned)
    hb, pb = host(b, pinned)
    hc, pc = host(c0.copy(), pinned)
    mask = rng.choice([0, 0, 0, 3, 5, 15])  # several bits: logical devices on the one GPU
    os.environ["BMMGPU_LOGICAL_DEVICES"] = "4"
    opts = bmm._opts(kernel, accumulate=accumulate, device_budget=budget, force_streaming=mode, device_mask=mask)
    st = lib.bmmgpu_cubic(pa, pb, pc, m, k, n, ring, ctypes.byref(opts))
    case = {"kind": "cubic", "m": m, "k": k, "n": n, "ring": ring, "kernel": kernel, "mode": mode, "budget": budget,
            "pinned": pinned, "accumulate": accumulate, "device_mask": mask}
    if st != 0:
        msg = lib.bmmgpu_last_error().decode()
        # a budget below the smallest out-of-core plan is a legitimate refusal
        if "exceed the device budget" in msg or "budget" in msg:
            return None
        return {**case, "status": st, "error": msg}
    got = words_of(hc)
    if not np.array_equal(got, want):
        bad = int(np.count_nonzero(got != want))
        return {**case, "mismatched_words": bad}
    return None


def alt_case(i: int) -> dict | None:
    n = rng.choice([256, 512, 1024, 2048, 4096])
    algo = rng.choice([1, 2, 3])
    depth = (n // 64).bit_length() - 1
    leaf = rng.choice([0, 6, 7, 8, 9, 10, 11, 12])
    if leaf and (1 << leaf) > n:
        leaf = 0
    pinned = rng.random() < 0.5
    a = orc.random(n, n, 5000 + i)
    b = orc.random(n, n, 6000 + i)
    want = orc.multiply_cubic(a, b, n, n, n, 1)
    ha, pa = host(a, pinned)
    hb, pb = host(b, pinned)
    hc, pc = host(np.zeros(n * n // 64, dtype=np.uint64), pinned)
    ds = rng.randint(0, depth)
    mask = rng.choice([0, 0, 3, 15])  # several bits: sub-instances dealt over logical devices
    dh = rng.randint(0, min(2, depth)) if mask else 0
    ds = min(ds, depth - dh)
    plan = bmm._Plan(dh, ds, depth - ds - dh, 1, 1)
    os.environ["BMMGPU_LOGICAL_DEVICES"] = "4"
    # overlapped leaf groups: off / 1-2 reserved pairs, both pass orders, groups down to 1 leaf
    ov, order, gmin = rng.choice(["0", "1", "1", "2"]), rng.choice(["0", "1"]), rng.choice(["1", "49", "343"])
    os.environ.update({"BMMGPU_ALT_OVERLAP": ov, "BMMGPU_ALT_OVERLAP_ORDER": order, "BMMGPU_ALT_OVERLAP_MIN": gmin})
    # out of core (force_streaming): one device -> the sub-instance driver, several -> tiles
    ooc = rng.random() < 0.3 and n >= 512
    opts = bmm._opts(0, leaf_log2=leaf, device_mask=mask, force_streaming=ooc)
    st = lib.bmmgpu_multiply(pa, pb, pc, n, algo, ctypes.byref(plan), 1, ctypes.byref(opts))
    case = {"kind": "alt", "n": n, "algo": algo, "leaf": leaf, "plan": [dh, ds, depth - ds - dh], "pinned": pinned,
            "device_mask": mask, "ooc": ooc, "overlap": [ov, order, gmin]}
    if st != 0:
        return {**case, "status": st, "error": lib.bmmgpu_last_error().decode()}
    if not np.array_equal(words_of(hc), want):
        return {**case, "mismatched_words": int(np.count_nonzero(words_of(hc) != want))}
    return None


t0 = time.time()
done = fails = 0
i = 0
while time.time() - t0 < budget_s:
    i += 1
    f = cubic_case(i) if rng.random() < 0.75 else alt_case(i)
    done += 1
    if f:
        fails += 1
        print(json.dumps(f), flush=True)
print(json.dumps({"cases": done, "failures": fails, "seconds": round(time.time() - t0, 1), "seed": seed}), flush=True)
sys.exit(1 if fails else 0)
