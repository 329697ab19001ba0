"""Per-step stage times of the 4M bench pipeline next to the same TRSM run
standalone on the pipeline's own A and R_s (is the in-pipeline TRSM slower?)."""
import json, os, sys
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch
sys.path.insert(0, ".")
import paper_2603_16644_b200 as sq
from paper_2603_16644_b200 import dense as D
from paper_2603_16644_b200.probgen import generate_problem_device

m, n = (int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22), 2048
dev = torch.device("cuda")
a, b, x_star = generate_problem_device(m, n, 10.0, 1e-6, 20261018, dev)
torch.cuda.synchronize()
rep = None
for i in range(4):
    rep = sq.algorithm1_pipeline(a, b, method="hpne", precision="auto", seed=1, x_star=x_star, diagnostics=False,
                                 stage_timing=True)
    print(json.dumps({"step": i, **{k: round(v, 1) for k, v in rep.stage_ms.items()}}))
r_s = rep.preconditioner.r_device()
if os.environ.get("PIPELINE_ONLY"):
    sys.exit(0)
sq.release_scratch()


def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); out = fn(); e.record(); e.synchronize()
        ts.append(round(s.elapsed_time(e), 1))
        del out
    return ts


print(json.dumps({"trsm_standalone_pipeline_R": timeit(lambda: D._trsm(a, r_s))}))
g = torch.Generator(device="cuda"); g.manual_seed(1)
r_rand = torch.triu(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)) + 8 * torch.eye(
    n, dtype=torch.float64, device="cuda")
print(json.dumps({"trsm_standalone_random_R": timeit(lambda: D._trsm(a, r_rand))}))
ap = D._trsm(a, r_s)
fin = torch.isfinite(ap).all().item()
print(json.dumps({"ap_finite": bool(fin), "ap_absmax": float(ap.abs().max()),
                  "ap_tiny_frac": float(((ap.abs() < 2.2e-308) & (ap != 0)).double().mean())}))
