"""Cost of page-locking host memory on this box: cudaMallocHost / cudaFreeHost
and cudaMalloc / cudaFree of 1-64 MB, alone (ctypes on the CUDA runtime)."""
import ctypes as C
import glob
import json
import time

import torch

torch.cuda.init()
torch.zeros(1, device="cuda")
lib = None
for p in sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*")) + ["libcudart.so.12"]:
    try:
        lib = C.CDLL(p)
        break
    except OSError:
        pass
res = {}
for mb in (1, 2, 4, 16, 64):
    n = mb << 20
    ptr = C.c_void_p()
    t0 = time.perf_counter(); lib.cudaMallocHost(C.byref(ptr), C.c_size_t(n)); t1 = time.perf_counter()
    C.memset(ptr, 1, n); t2 = time.perf_counter()
    lib.cudaFreeHost(ptr); t3 = time.perf_counter()
    d = C.c_void_p()
    t4 = time.perf_counter(); lib.cudaMalloc(C.byref(d), C.c_size_t(n)); t5 = time.perf_counter()
    lib.cudaFree(d); t6 = time.perf_counter()
    res[f"{mb}MB"] = {k: round(1e3 * v, 3) for k, v in dict(mallochost=t1 - t0, touch=t2 - t1, freehost=t3 - t2,
                                                              malloc=t5 - t4, free=t6 - t5).items()}
print(json.dumps(res))
