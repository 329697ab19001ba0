"""Time sk_lu_solve_f64 (n x n, partial pivoting) for a grid-size override SK_LU_BLOCKS
given on the command line (the env is read once per process): CUDA events, best of 5."""
import json, os, sys
os.environ["SK_LU_BLOCKS"] = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("SK_LU_BLOCKS", "296")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_16644_b200 import dense

n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
rhs = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
x0 = dense._lu_solve(a, rhs)
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); x = dense._lu_solve(a, rhs); e.record(); e.synchronize()
    ts.append(s.elapsed_time(e))
assert torch.equal(x, x0)
print(json.dumps({"blocks": os.environ["SK_LU_BLOCKS"], "n": n, "ms_best": min(ts), "ms": ts,
                  "x_sum": float(x.sum())}))
