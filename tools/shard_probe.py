"""The row-sharded pipeline (what bench.py runs on every rank under torchrun) timed on
one GPU next to algorithm1_pipeline: per-rank cost of the weak-scaled solve."""
import json, os, sys
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch
sys.path.insert(0, ".")
import paper_2603_16644_b200 as sq
from paper_2603_16644_b200.distributed import algorithm1_pipeline_sharded
from paper_2603_16644_b200.probgen import generate_problem_device

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
n = 2048
a, b, x_star = generate_problem_device(m, n, 10.0, 1e-6, 20261018, torch.device("cuda"))
torch.cuda.synchronize()
for name, fn in (("pipeline", lambda: sq.algorithm1_pipeline(a, b, method="hpne", precision="auto", seed=1,
                                                               x_star=x_star, diagnostics=False, stage_timing=True)),
                 ("sharded", lambda: algorithm1_pipeline_sharded(a, b, method="hpne", precision="auto", seed=1,
                                                                 x_star=x_star, stage_timing=True))):
    fn(); fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    reps = [fn() for _ in range(3)]
    e.record(); e.synchronize()
    r = reps[-1]
    print(json.dumps({"impl": name, "ms": round(s.elapsed_time(e) / 3, 1), "rel_error": r.relative_error,
                      "level": r.preconditioner.computed_in.name,
                      "stages": {k: round(v, 1) for k, v in r.stage_ms.items()}}))
