"""cudaHostRegister cost and H2D bandwidth straight from a registered pageable numpy buffer
(the alternative to staging pageable input through a pinned ring)."""
import ctypes, json, time
import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so") if False else None
from cuda.bindings import runtime as rt   # cuda-python
out = {}
for gb in (1, 4):
    n = gb * 2**30 // 8
    a = np.ones(n)                                 # pageable, touched
    ptr = a.ctypes.data
    t = time.perf_counter()
    err, = rt.cudaHostRegister(ptr, a.nbytes, 0)
    out[f"register_{gb}GiB_s"] = time.perf_counter() - t
    out[f"register_{gb}GiB_err"] = int(err)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    h = torch.from_numpy(a)
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(h, non_blocking=True); e.record(); e.synchronize()
    out[f"h2d_registered_{gb}GiB_GBs"] = a.nbytes / (s.elapsed_time(e) / 1e3) / 1e9
    t = time.perf_counter()
    rt.cudaHostUnregister(ptr)
    out[f"unregister_{gb}GiB_s"] = time.perf_counter() - t
    del d
print(json.dumps(out))
