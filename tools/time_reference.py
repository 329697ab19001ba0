"""Time the SHIPPED reference (`sketchlsq` 0.1.0 from /root/reference, diagnostics as
shipped) on this container's host cores, as SURVEY §8(d)'s CPU-baseline row asks:
config 1 (generate_problem(1000, 100, 1e8, rho), HPNE "single", 3 trials per rho),
config 2 (100000 x 1000, kappa 1e10, rho 1e-6, PNE and HPNE sharing one fixed binary32
preconditioner; the problem is drawn with the LAPACK generator of oracle/problems.py
because the reference's own Householder generator needs far too long at this size) and
the ladder 6000 x 100, 20000 x 250, 50000 x 500 (algorithm1_pipeline pne auto) with a
fit t = c m n^2.  Build container only (needs /root/reference); writes one JSON document.

    python tools/time_reference.py > profiles/r2_reference_cpu_timings.json
"""
import json
import os
import platform
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import sketchlsq as sq
    from threadpoolctl import threadpool_info

    from oracle.problems import planted_problem_lapack
    out = {"reference": "sketchlsq " + sq.__version__, "host": platform.processor() or platform.machine(),
           "cpu_count": os.cpu_count(),
           "blas": [{k: i.get(k) for k in ("internal_api", "num_threads", "version")} for i in threadpool_info()],
           "note": "build container's host (not the GPU box's 16 cores)"}

    def timed(fn):
        t = time.perf_counter()
        r = fn()
        return r, time.perf_counter() - t

    # config 1
    c1 = []
    for rho in (1e-12, 1e-6, 1e-2):
        for trial in range(3):
            seed = sq.rng.mix64(20261019, int(-np.log10(rho)), trial)
            p = sq.generate_problem(1000, 100, 1e8, rho, seed)
            try:
                rep, s = timed(lambda: sq.algorithm1_pipeline(p.a, p.b, "hpne", "single", 3.0, "dct2", seed, p.x_star))
                c1.append({"rho": rho, "trial": trial, "seconds": s, "rel_error": rep.relative_error,
                           "kappa_rs": rep.preconditioner.kappa_rs})
            except sq.SketchLsqError as ex:
                c1.append({"rho": rho, "trial": trial, "error": type(ex).__name__})
    ok = [r["seconds"] for r in c1 if "seconds" in r]
    out["config1"] = {"runs": c1, "median_seconds": float(np.median(ok)) if ok else None}

    # config 2 (as shipped the kappa(R_s) diagnostic runs inside build_preconditioner; at
    # kappa 1e10 its Jacobi may not converge: the outcome is recorded)
    def attempt(fn):
        t = time.perf_counter()
        try:
            return "ok", fn(), time.perf_counter() - t
        except sq.SketchLsqError as ex:
            return type(ex).__name__, None, time.perf_counter() - t

    p = planted_problem_lapack(100000, 1000, 1e10, 1e-6, 20261019)
    c2 = {}
    o, pre, s = attempt(lambda: sq.build_preconditioner(p.a, 3.0, "dct2", sq.BINARY32, 0))
    c2["build_preconditioner"] = {"outcome": o, "seconds": s}
    if pre is not None:
        o, ap, s = attempt(lambda: sq.precondition_matrix(p.a, pre))
        c2["precondition_matrix"] = {"outcome": o, "seconds": s}
        if ap is not None:
            for name, fn in (("solve_pne", sq.solve_pne), ("solve_hpne", sq.solve_hpne)):
                o, rep, s = attempt(lambda: fn(p.a, p.b, pre, x_star=p.x_star, a_p=ap))
                c2[name] = {"outcome": o, "seconds": s, "rel_error": rep.relative_error if rep else None}
    o, rep, s = attempt(lambda: sq.algorithm1_pipeline(p.a, p.b, "pne", "single", 3.0, "dct2", 0, p.x_star))
    c2["algorithm1_pipeline_pne_single"] = {"outcome": o, "seconds": s,
                                            "rel_error": rep.relative_error if rep else None}
    out["config2"] = c2

    # ladder
    ladder = []
    for m, n in ((6000, 100), (20000, 250), (50000, 500)):
        p = planted_problem_lapack(m, n, 1e4, 1e-6, m + n)
        o, rep, s = attempt(lambda: sq.algorithm1_pipeline(p.a, p.b, "pne", "auto", 3.0, "dct2", 1, p.x_star))
        ladder.append({"m": m, "n": n, "seconds": s, "outcome": o,
                       "level": rep.preconditioner.computed_in.name if rep else None,
                       "rel_error": rep.relative_error if rep else None})
    mn2 = np.array([r["m"] * r["n"] ** 2 for r in ladder], dtype=float)
    ts = np.array([r["seconds"] for r in ladder])
    c = float((mn2 @ ts) / (mn2 @ mn2))
    out["ladder"] = {"runs": ladder, "fit_c_seconds_per_mn2": c,
                     "fit_residual_rel": [float(t / (c * x) - 1) for t, x in zip(ts, mn2)],
                     "config3_extrapolated_seconds": c * 4194304 * 2048 ** 2,
                     "config3_note": "not run: A alone is 68.7 GB and the reference's column loops would take "
                                     "about this long by the fitted model"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
