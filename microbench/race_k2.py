"""K2 (cubic_umma2_kernel) under compute-sanitizer: a batch of short-K GF(2) and Boolean
products with more tiles than CTA pairs (every pair hands its accumulator over several
times), checked bit-exactly against the oracle.  Dev helper for the race investigation:

    compute-sanitizer --tool racecheck python microbench/race_k2.py [batch] [L] [K]
"""
from __future__ import annotations

import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_01554_b200 as bmm  # noqa: E402
from oracle import Oracle  # noqa: E402  (checker only)


def main() -> None:
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 160
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
    lib = bmm.lib()
    orc = Oracle()
    kw = K // 64
    g = torch.Generator().manual_seed(7)
    hA = torch.randint(-2**62, 2**62, (batch, L, kw), dtype=torch.int64, generator=g)
    hBt = torch.randint(-2**62, 2**62, (batch, L, kw), dtype=torch.int64, generator=g)
    dA, dBt = hA.cuda(), hBt.cuda()
    dC = torch.empty((batch, L, L // 64), dtype=torch.int64, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    bad = 0
    for ring in (1, 0):
        st = lib.bmmgpu_dev_cubic_batched(dA.data_ptr(), kw, L * kw, dBt.data_ptr(), kw, L * kw, dC.data_ptr(),
                                          L // 64, L * (L // 64), batch, L, L, kw, ring, 2, 0, sp)
        assert st == 0, lib.bmmgpu_last_error()
        torch.cuda.synchronize()
        got = dC.cpu().numpy().view(np.uint64)
        for b in range(0, batch, max(1, batch // 8)):
            a = hA[b].numpy().view(np.uint64).ravel()
            # oracle takes row-major B: B = Bt^T via transpose of the bit matrix
            bt_bits = np.unpackbits(hBt[b].numpy().view(np.uint8), axis=1, bitorder="little")  # L x K
            B = np.packbits(bt_bits.T.copy(), axis=1, bitorder="little").view(np.uint64).ravel()
            want = orc.multiply_cubic(a, B, L, K, L, ring)
            if not np.array_equal(want, got[b].ravel()):
                bad += 1
                print(f"MISMATCH ring={ring} product={b}")
    print(f"race_k2 batch={batch} L={L} K={K}: {'OK' if bad == 0 else f'{bad} mismatches'}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
