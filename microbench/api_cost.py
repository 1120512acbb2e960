"""Host cost of the CUDA runtime calls a bmmgpu_cubic call makes (dev helper)."""
import json
import time

import torch
from cuda.bindings import runtime as rt

torch.cuda.init()
torch.empty(1, device="cuda")


def cost(name, fn, reps=200):
    for _ in range(10):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    print(json.dumps({"call": name, "us": round((time.perf_counter() - t0) / reps * 1e6, 2)}), flush=True)


cost("cudaMemGetInfo", lambda: rt.cudaMemGetInfo())
cost("cudaGetDeviceCount", lambda: rt.cudaGetDeviceCount())
cost("cudaSetDevice", lambda: rt.cudaSetDevice(0))
cost("cudaDeviceGetAttribute(SMs)", lambda: rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMultiProcessorCount, 0))


def stream_cd():
    _, s = rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)
    rt.cudaStreamDestroy(s)


cost("cudaStreamCreate+Destroy", stream_cd)


def event_cd():
    _, e = rt.cudaEventCreateWithFlags(rt.cudaEventDisableTiming)
    rt.cudaEventDestroy(e)


cost("cudaEventCreate+Destroy", event_cd)
_, s = rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)


def malloc_async():
    _, p = rt.cudaMallocAsync(8 << 20, s)
    rt.cudaFreeAsync(p, s)


cost("cudaMallocAsync+FreeAsync 8MiB", malloc_async)
cost("cudaStreamSynchronize(idle)", lambda: rt.cudaStreamSynchronize(s))
h = torch.empty(1 << 20, dtype=torch.int64, pin_memory=True)
cost("cudaPointerGetAttributes", lambda: rt.cudaPointerGetAttributes(h.data_ptr()))
d = torch.empty(1 << 10, dtype=torch.int64, device="cuda")


def tiny_copy_sync():
    rt.cudaMemcpyAsync(d.data_ptr(), h.data_ptr(), 8192, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s)
    rt.cudaStreamSynchronize(s)


cost("8 KiB H2D + sync", tiny_copy_sync)
