"""Achievable INT8 tensor throughput on this B200 (cuBLASLt via torch._int_mm),
the denominator for an INT8-emulated FP64 Gram."""
import json
import torch

out = {}
for (m, k, n) in [(8192, 8192, 8192), (2048, 131072, 2048), (4096, 65536, 4096)]:
    a = torch.randint(-127, 127, (m, k), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 127, (n, k), dtype=torch.int8, device="cuda").t()
    torch._int_mm(a, b); torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); torch._int_mm(a, b); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    out[f"{m}x{k}x{n}"] = {"ms": round(best, 3), "tops": round(2 * m * n * k / (best * 1e-3) / 1e12, 1)}
print(json.dumps(out))
