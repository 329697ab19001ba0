"""Per-solve latency at configs 1 and 2 (small, launch/latency-bound): wall time per
algorithm1_pipeline call from numpy (the reference's convention) and from device
tensors, with the number of libsklsq kernel launches and host synchronisations.

    python tools/latency_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200 import _lib
    from oracle.problems import planted_problem
    lib = _lib.lib()
    cases = {"config1": (1000, 100, 1e8, 1e-6, "hpne", "single"),
             "config2": (100000, 1000, 1e10, 1e-6, "pne", "single")}
    for name, (m, n, kappa, rho, method, prec) in cases.items():
        if name == "config2":
            from paper_2603_16644_b200.probgen import generate_problem_device
            a_d, b_d, xs = generate_problem_device(m, n, kappa, rho, 3)
            a_np, b_np, xs_np = a_d.cpu().numpy(), b_d.cpu().numpy(), xs.cpu().numpy()
        else:
            p = planted_problem(m, n, kappa, rho, 11)
            a_np, b_np, xs_np = p.a, p.b, p.x_star
            a_d, b_d = torch.from_numpy(a_np).cuda(), torch.from_numpy(b_np).cuda()
        out = {"case": name, "m": m, "n": n, "kappa": kappa, "method": method, "precision": prec}
        for kind, (a, b) in {"numpy": (a_np, b_np), "device": (a_d, b_d)}.items():
            for _ in range(3):
                sq.algorithm1_pipeline(a, b, method=method, precision=prec, seed=1, diagnostics=False)
            torch.cuda.synchronize()
            reps = 20
            l0 = lib.sk_launch_count()
            t = time.perf_counter()
            for _ in range(reps):
                rep = sq.algorithm1_pipeline(a, b, method=method, precision=prec, seed=1, x_star=xs_np,
                                             diagnostics=False)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t) / reps
            out[kind] = {"ms_per_solve": dt * 1e3, "launches_per_solve": (lib.sk_launch_count() - l0) / reps,
                         "rel_error": rep.relative_error, "level": rep.preconditioner.computed_in.name}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
