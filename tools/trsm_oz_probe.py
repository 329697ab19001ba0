"""Blocked INT8-update TRSM against the one-kernel DMMA TRSM at m x n (default 4M x 2048):
CUDA-event times, the max difference and the backward residual on a row sample."""
import json, sys
import torch
sys.path.insert(0, ".")
from paper_2603_16644_b200 import dense as D
from paper_2603_16644_b200 import _lib

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
g = torch.Generator(device="cuda"); g.manual_seed(1)
a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
r = torch.triu(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)) + 8 * torch.eye(
    n, dtype=torch.float64, device="cuda")
o = torch.empty_like(a)
sample = {}
rows = slice(0, min(m, 262144))
for eng in ("dmma", "ozaki"):
    D._trsm(a, r, out=o, engine=eng); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); D._trsm(a, r, out=o, engine=eng); e.record(); e.synchronize()
        ts.append(round(s.elapsed_time(e), 1))
    sample[eng] = o[rows].clone()
    print(json.dumps({"engine": eng, "m": m, "n": n, "ms": ts,
                      "fell_back": _lib.lib().sk_trsm_ozaki_fell_back() if eng == "ozaki" else None}), flush=True)
d = (sample["ozaki"] - sample["dmma"]).abs().max().item() / sample["dmma"].abs().max().item()
res = {k: ((v @ r - a[rows]).norm() / (v.norm() * r.norm())).item() for k, v in sample.items()}
print(json.dumps({"max_rel_diff": d, "backward_sample": res}))
