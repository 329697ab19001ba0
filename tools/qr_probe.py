"""Time sk_qr_r on a d x n sketch at a level (CUDA events around the device call, best
of 5); SK_QR_SMEM=0 in the environment selects the global-memory flow kernel."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_16644_b200 import dense

d, n, level = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dt = {16: torch.float16, 32: torch.float32, 64: torch.float64}[level]
g = torch.Generator(device="cuda").manual_seed(3)
a = torch.randn(n, d, dtype=torch.float64, device="cuda", generator=g).to(dt)   # column-major d x n
r0 = dense._qr_r(a.clone(), level, d, n)
ts = []
for _ in range(5):
    w = a.clone()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); r = dense._qr_r(w, level, d, n); e.record(); e.synchronize()
    ts.append(s.elapsed_time(e))
assert torch.equal(r, r0)
print(json.dumps({"d": d, "n": n, "level": level, "smem": os.environ.get("SK_QR_SMEM", "default"),
                  "ms_best": min(ts), "ms": ts}))
