"""TRSM at 4M x 2048 as the pipeline calls it (fresh padded A_p per call) vs a
preallocated padded / unpadded output."""
import json, os, sys
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch
sys.path.insert(0, ".")
from paper_2603_16644_b200 import dense as D

m, n = 1 << 22, 2048
g = torch.Generator(device="cuda"); g.manual_seed(1)
a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
r = torch.triu(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)) + 8 * torch.eye(
    n, dtype=torch.float64, device="cuda")


def timeit(fn, reps=4):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); out = fn(); e.record(); e.synchronize()
        ts.append(round(s.elapsed_time(e), 1))
        del out
    return ts


print(json.dumps({"fresh_padded": timeit(lambda: D._trsm(a, r))}))
buf = torch.empty((m, n + 8), dtype=torch.float64, device="cuda")[:, :n]
print(json.dumps({"prealloc_padded": timeit(lambda: D._trsm(a, r, out=buf))}))
del buf
torch.cuda.empty_cache()
buf = torch.empty((m, n), dtype=torch.float64, device="cuda")
print(json.dumps({"prealloc_unpadded": timeit(lambda: D._trsm(a, r, out=buf))}))
