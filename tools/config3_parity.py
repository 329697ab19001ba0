"""Config-3 parity at FULL size (4,194,304 x 2048) against the row-chunked hybrid CPU
oracle (oracle/hybrid.py), for the three kappa points of SURVEY §8(d) config 3.

Per kappa: one planted problem on the GPU (probgen.generate_problem_device), the GPU
solve (algorithm1_pipeline, precision="auto"), the same A and b copied to the host and
solved by the hybrid oracle, and the reference estimator (restatement of
estimate_log10_condition, src/precision.py:205-251) run on the planted n x n R
(A^T A = R^T R).  Writes one JSON line per (kappa, method) to stdout.

    python tools/config3_parity.py [--m 4194304] [--kappas 10,1e3,2e6] [--methods hpne,pne]
"""
import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4 * 1024 * 1024)
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--kappas", default="10,1e3,2e6")
    ap.add_argument("--methods", default="hpne,pne")
    ap.add_argument("--seed", type=int, default=20261018)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2603_16644_b200 as sq
    from oracle import hybrid
    from oracle import restatement as R
    from paper_2603_16644_b200.probgen import generate_problem_device, planted_triangle_device

    for kappa in [float(k) for k in args.kappas.split(",")]:
        a, b, xs = generate_problem_device(args.m, args.n, kappa, 1e-6, args.seed)
        r = planted_triangle_device(args.n, kappa, args.seed + 1).cpu().numpy()
        k0_r, over_r = R.kappa0_from_gram(r.T @ r)
        ah, bh, xh = a.cpu().numpy(), b.cpu().numpy(), xs.cpu().numpy()
        for method in args.methods.split(","):
            torch.cuda.synchronize()
            t = time.perf_counter()
            got = sq.algorithm1_pipeline(a, b, method=method, precision="auto", seed=1, x_star=xs,
                                         diagnostics=False)
            torch.cuda.synchronize()
            gpu_s = time.perf_counter() - t
            tm = {}
            t = time.perf_counter()
            ref = hybrid.pipeline(ah, bh, method=method, precision="auto", seed=1, x_star=xh, timings=tm)
            cpu_s = time.perf_counter() - t
            line = {
                "m": args.m, "n": args.n, "kappa": kappa, "method": method,
                "reference_estimator_on_R": {"kappa0": k0_r, "overflowed": over_r,
                                             "level": R.choose_level(k0_r, over_r)},
                "oracle": {"kappa0": ref.decision[0], "level": ref.pre.level, "escalated_from": ref.escalated_from,
                           "rel_error": ref.relative_error, "rel_residual": ref.relative_residual,
                           "seconds": cpu_s, "stages_s": tm},
                "gpu": {"kappa0": got.precision_decision.kappa0, "level": got.preconditioner.computed_in.name,
                        "escalated_from": got.escalated_from.name if got.escalated_from else None,
                        "rel_error": got.relative_error, "rel_residual": got.relative_residual,
                        "seconds_first_call": gpu_s},
            }
            line["same_level"] = line["oracle"]["level"] == line["gpu"]["level"] == \
                line["reference_estimator_on_R"]["level"]
            line["same_escalation"] = line["oracle"]["escalated_from"] == line["gpu"]["escalated_from"]
            line["error_ratio_gpu_over_oracle"] = got.relative_error / ref.relative_error
            line["gate_ok"] = bool(line["same_level"] and line["same_escalation"] and
                                   got.relative_error <= max(10 * ref.relative_error, 1e-14))
            print(json.dumps(line), flush=True)
        del a, b, ah, bh
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
