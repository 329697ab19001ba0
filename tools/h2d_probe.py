"""Host<->device copy bandwidth from pinned / pageable host memory (context for e2e)."""
import json, time, torch
out = {}
for gb in (1, 8):
    n = gb * 2**30 // 8
    t0 = time.time(); h = torch.empty(n, dtype=torch.float64, pin_memory=True); out[f"pin_alloc_{gb}GiB_s"] = time.time() - t0
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(h, non_blocking=True); e.record(); e.synchronize()
    out[f"h2d_pinned_{gb}GiB_GBs"] = gb * 2**30 / (s.elapsed_time(e) / 1e3) / 1e9
    s.record(); h.copy_(d, non_blocking=True); e.record(); e.synchronize()
    out[f"d2h_pinned_{gb}GiB_GBs"] = gb * 2**30 / (s.elapsed_time(e) / 1e3) / 1e9
    p = torch.empty(n, dtype=torch.float64); p.fill_(1.0)
    s.record(); d.copy_(p); e.record(); e.synchronize()
    out[f"h2d_pageable_{gb}GiB_GBs"] = gb * 2**30 / (s.elapsed_time(e) / 1e3) / 1e9
    del h, d, p
print(json.dumps(out))
