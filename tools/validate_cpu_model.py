"""Validate bench.py's CPU reference model (m-linear stages timed on a full-n row slice
and scaled in m) against the same stages measured at a larger full height.

    python tools/validate_cpu_model.py [--m 524288] [--slice 8192] [--n 2048]

Prints one JSON line: per stage the slice-scaled prediction, the measured time at m, and
their ratio.  The m-independent stages are timed at full size in both and are not part
of the check."""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def stages(a, b, level, seed=1):
    import numpy as np
    from oracle import restatement as R
    m, n = a.shape
    d = 3 * n
    t = {}
    t0 = time.perf_counter(); a.T @ a; t["kappa0_gram"] = time.perf_counter() - t0
    data, _ = R.demote(a, level)
    op = R.draw_sketch(m, d, "dct2", seed)
    t0 = time.perf_counter(); R.sketch_apply(op, data); t["sketch"] = time.perf_counter() - t0
    del data
    r = np.triu(np.random.default_rng(3).standard_normal((n, n))) + n * np.eye(n)
    t0 = time.perf_counter(); ap = np.ascontiguousarray(R.tri_solve(r, a.T, transposed=True).T)
    t["trsm"] = time.perf_counter() - t0
    t0 = time.perf_counter(); ap.T @ a, ap.T @ b; t["gram"] = time.perf_counter() - t0
    del ap
    x = np.ones(n)
    t0 = time.perf_counter(); np.linalg.norm(a @ x - b); t["report"] = time.perf_counter() - t0
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=524288)
    ap.add_argument("--slice", type=int, default=8192)
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--level", default="binary16")
    args = ap.parse_args()
    import numpy as np
    rng = np.random.default_rng(12345)
    cols = 10.0 ** (-np.arange(args.n) / max(args.n - 1, 1))
    big = rng.standard_normal((args.m, args.n)) * cols[None, :]
    bb = rng.standard_normal(args.m)
    small, sb = big[: args.slice].copy(), bb[: args.slice].copy()
    ts = stages(small, sb, args.level)
    scale = {k: args.m / args.slice for k in ts}
    scale["sketch"] = (args.m * math.log2(args.m)) / (args.slice * math.log2(args.slice))
    pred = {k: ts[k] * scale[k] for k in ts}
    tm = stages(big, bb, args.level)
    out = {"m": args.m, "slice": args.slice, "n": args.n, "level": args.level, "threads": os.cpu_count(),
           "slice_s": ts, "predicted_s": pred, "measured_s": tm,
           "ratio_measured_over_predicted": {k: tm[k] / pred[k] for k in tm},
           "total_predicted_s": sum(pred.values()), "total_measured_s": sum(tm.values())}
    out["total_ratio"] = out["total_measured_s"] / out["total_predicted_s"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
