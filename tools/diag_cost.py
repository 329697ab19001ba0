"""Cost of the default API (diagnostics=True: kappa(R_s) and kappa(A_p) filled like the
reference's src/solvers.py:200, :214) against diagnostics=False, at config 2
(100000 x 1000, kappa 1e10, fixed single) and config 3 (4M x 2048, auto).

    python tools/diag_cost.py [--configs 2,3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3")
    args = ap.parse_args()
    import torch
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200.probgen import generate_problem_device
    cfg = {"2": (100000, 1000, 1e10, "single", "pne"), "3": (4 * 1024 * 1024, 2048, 10.0, "auto", "hpne")}
    for c in args.configs.split(","):
        m, n, kappa, prec, method = cfg[c]
        a, b, xs = generate_problem_device(m, n, kappa, 1e-6, 7)
        out = {"config": c, "m": m, "n": n, "kappa": kappa, "precision": prec, "method": method}
        for diag in (False, True, False, True):
            torch.cuda.synchronize()
            t = time.perf_counter()
            rep = sq.algorithm1_pipeline(a, b, method=method, precision=prec, seed=1, x_star=xs, diagnostics=diag,
                                         stage_timing=True)
            torch.cuda.synchronize()
            key = "diagnostics_on" if diag else "diagnostics_off"
            out[key] = {"ms": (time.perf_counter() - t) * 1e3, "wall_ms": rep.wall_ms,
                        "kappa_rs": rep.preconditioner.kappa_rs, "kappa_ap": rep.preconditioner.kappa_ap,
                        "rel_error": rep.relative_error,
                        "diag_ms": {k: v for k, v in rep.stage_ms.items() if k.startswith("diag")}}
        print(json.dumps(out), flush=True)
        del a, b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
