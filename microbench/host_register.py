"""Cost of page-locking a caller's pageable buffer for one call (cudaHostRegister +
cudaHostUnregister) against the size, to decide how the drop-in should move std::vector
storage (dev helper)."""
import ctypes
import json
import time

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so")
torch.zeros(1, device="cuda")
for mib in (64, 512, 2048):
    a = np.ones(mib << 17, dtype=np.uint64)  # touched
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        assert cudart.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 0) == 0
        t1 = time.perf_counter()
        assert cudart.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data)) == 0
        t2 = time.perf_counter()
        ts.append((t1 - t0, t2 - t1))
    print(json.dumps({"MiB": mib, "register_s": [round(x[0], 4) for x in ts], "unregister_s": [round(x[1], 4) for x in ts],
                      "register_GBps": round(a.nbytes / min(x[0] for x in ts) / 1e9, 1)}), flush=True)
