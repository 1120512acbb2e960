"""Multi-device fast GF(2) product: the top host levels of the recursion
are dealt across devices as independent sub-instances (the reference host layer,
pipeline.cpp:198-369, on devices) and the partial products are XOR-folded slab by slab.
Only one GPU is reachable here, so the multi-device runs use the BMMGPU_LOGICAL_DEVICES
test hook: k logical devices, each with its own host thread, buffers and peer copies,
mapped onto the physical GPU."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import HAS_GPU

GF2 = 1


def test_host_level_choice_is_the_most_even_deal():
    """Pure host arithmetic (no device): the smallest dh whose round-robin deal of 7^dh
    sub-instances is within 3 % of even, sub-instances >= 8192, one level left below."""
    import paper_1909_01554_b200 as bmm
    lib = bmm.lib()
    assert lib.bmmgpu_host_levels(262144, 1, 0) == 0
    assert lib.bmmgpu_host_levels(262144, 7, 0) == 1      # 7 over 7: even
    assert lib.bmmgpu_host_levels(262144, 2, 0) == 2      # 25 of 49 on the busiest: 2 % over
    assert lib.bmmgpu_host_levels(262144, 8, 0) == 3      # 43 of 343 (42.9 even)
    assert lib.bmmgpu_host_levels(65536, 8, 0) == 3       # sub-instances of 8192
    assert lib.bmmgpu_host_levels(16384, 8, 0) == 1       # e = 2: one level must stay below


def _rand(oracle, n, seed):
    return oracle.random(n, n, seed)


@pytest.mark.gpu
@pytest.mark.skipif(not HAS_GPU, reason="no CUDA device")
@pytest.mark.parametrize("devices", [2, 3, 8])
def test_multiply_on_several_devices_matches_oracle(oracle, monkeypatch, devices):
    import paper_1909_01554_b200 as bmm
    monkeypatch.setenv("BMMGPU_LOGICAL_DEVICES", str(devices))
    lib = bmm.lib()
    n = 2048
    a, b = _rand(oracle, n, 701), _rand(oracle, n, 702)
    want = oracle.multiply_cubic(a, b, n, n, n, GF2)
    for algo in (1, 2, 3):
        for d_host in (0, 1, 2):
            c = np.zeros_like(a)
            plan = bmm._Plan(d_host, 0, 5 - d_host, 1, 1)
            opts = bmm._opts(0, leaf_log2=8, device_mask=(1 << devices) - 1)
            st = lib.bmmgpu_multiply(a.ctypes.data, b.ctypes.data, c.ctypes.data, n, algo, ctypes.byref(plan), GF2,
                                     ctypes.byref(opts))
            assert st == 0, lib.bmmgpu_last_error()
            assert np.array_equal(c, want), (algo, d_host)


@pytest.mark.gpu
@pytest.mark.skipif(not HAS_GPU, reason="no CUDA device")
@pytest.mark.parametrize("dh", [1, 2, 3])
def test_partial_products_xor_to_the_product(oracle, dh):
    """bmmgpu_dev_multiply_partial over any round-robin partition of the sub-instances:
    the XOR of the partials is the product; a single part is not (non-vacuous)."""
    import torch
    import paper_1909_01554_b200 as bmm
    lib = bmm.lib()
    n, leaf = 4096, 7
    w = n // 64
    a, b = _rand(oracle, n, 711 + dh), _rand(oracle, n, 721 + dh)
    want = oracle.multiply_cubic(a, b, n, n, n, GF2)
    dA = torch.from_numpy(a.view(np.int64)).view(n, w).cuda()
    dB = torch.from_numpy(b.view(np.int64)).view(n, w).cuda()
    dBt = torch.empty((n, w), dtype=torch.int64, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.bmmgpu_dev_transpose(dB.data_ptr(), w, n, n, dBt.data_ptr(), n, w, sp) == 0
    part = torch.empty_like(dA)
    for stride in (1, 3, 7, 50):
        acc = torch.zeros_like(dA)
        for first in range(stride):
            st = lib.bmmgpu_dev_multiply_partial(dA.data_ptr(), w, dBt.data_ptr(), w, part.data_ptr(), w, n, 2, dh,
                                                 first, stride, leaf, 0, sp)
            assert st == 0, lib.bmmgpu_last_error()
            if stride > 1 and first == 0:
                assert not np.array_equal(part.cpu().numpy().view(np.uint64).ravel(), want)
            acc ^= part
        assert np.array_equal(acc.cpu().numpy().view(np.uint64).ravel(), want), stride
    assert lib.bmmgpu_dev_multiply_partial(dA.data_ptr(), w, dBt.data_ptr(), w, part.data_ptr(), w, n, 2, 6, 0, 1,
                                           leaf, 0, sp) == 1  # no level left below the host levels
