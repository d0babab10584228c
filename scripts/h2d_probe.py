"""Dev probe: host<->device copy bandwidth for 4 MiB buffers from torch
pinned memory vs cudaHostAlloc(WriteCombined / Portable) memory, one at a
time and H2D + D2H concurrently on two streams."""
import ctypes as C
import time
import numpy as np
import torch
import cuda.bindings.runtime as rt

N = 4 << 20
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
dev2 = torch.empty(N, dtype=torch.uint8, device="cuda")


def host(flags):
    if flags is None:
        return torch.empty(N, dtype=torch.uint8).pin_memory()
    err, p = rt.cudaHostAlloc(N, flags)
    assert err == rt.cudaError_t.cudaSuccess
    arr = (C.c_uint8 * N).from_address(int(p))
    return torch.from_numpy(np.frombuffer(arr, np.uint8))


def bw(fn, n=50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return N * n / (time.perf_counter() - t0) / 1e9


for name, flags in (("torch pinned", None), ("hostalloc default", 0),
                    ("hostalloc WC", rt.cudaHostAllocWriteCombined),
                    ("hostalloc portable", rt.cudaHostAllocPortable)):
    h = host(flags)
    h2 = host(flags)
    h[:] = 1
    h2d = bw(lambda: dev.copy_(h, non_blocking=True))
    d2h = bw(lambda: h2.copy_(dev, non_blocking=True))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            dev.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(dev2, non_blocking=True)
    dual = bw(both)
    print(f"{name:20s}: H2D {h2d:5.1f} GB/s  D2H {d2h:5.1f} GB/s  concurrent (each) {dual:5.1f} GB/s")
