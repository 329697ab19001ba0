"""TRSM rate and run-to-run spread against the column count n at m = 4M rows
(is the left-looking re-read traffic what makes n = 2048 slow and noisy?)."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_2603_16644_b200 import dense as D

m = 1 << 22
g = torch.Generator(device="cuda"); g.manual_seed(1)
buf = torch.randn(m * 2048, dtype=torch.float64, device="cuda", generator=g)
out = torch.empty_like(buf)
for n in [int(x) for x in (sys.argv[1:] or ["2048", "1024", "512"])]:
    a = buf[: m * n].view(m, n)
    o = out[: m * n].view(m, n)
    r = torch.triu(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)) + 8 * torch.eye(
        n, dtype=torch.float64, device="cuda")
    D._trsm(a, r, out=o); torch.cuda.synchronize()
    ts = []
    for _ in range(6):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); D._trsm(a, r, out=o); e.record(); e.synchronize()
        ts.append(round(s.elapsed_time(e), 1))
    print(json.dumps({"n": n, "ms": ts, "tflops_best": round(m * n * n / (min(ts) * 1e-3) / 1e12, 2),
                      "tflops_worst": round(m * n * n / (max(ts) * 1e-3) / 1e12, 2)}))
