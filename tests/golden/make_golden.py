"""Generate golden fixtures by running the REAL reference (`sketchlsq` 0.1.0).

Run in the build container only (needs /root/reference, which the GPU box does
not have):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/golden.npz (+ golden_meta.json).  Problems are stored by
seed plus a SHA-256 of the generated A/b bytes; the oracle regenerates them and
the tests check the hash, which pins `oracle.problems` bitwise.  A few small
matrices are stored in full.
"""
import hashlib
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import sketchlsq as sq  # noqa: E402
from sketchlsq.precision import _pairwise_sum  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
arrays = {}
meta = {"reference": "sketchlsq " + sq.__version__, "cases": {}}


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def outcome(fn):
    try:
        return fn(), None
    except sq.SketchLsqError as ex:
        return None, type(ex).__name__


def put(key, value):
    arrays[key] = np.asarray(value)


# 1. planted problems: hashes (+ full arrays for the small ones)
PROBLEMS = {
    "p600_k1e2": (600, 40, 1e2, 1e-8, 4),
    "p600_k1e6": (600, 40, 1e6, 1e-8, 4),
    "p600_k1e10": (600, 40, 1e10, 1e-8, 4),
    "p600_k1e6_s6": (600, 40, 1e6, 1e-8, 6),
    "p600_k1e2_s3": (600, 40, 1e2, 1e-8, 3),
    "p300_k10_s5": (300, 20, 10.0, 1e-4, 5),
    "p250_k1e2_s7": (250, 18, 1e2, 1e-6, 7),
    "p200_k1e3_s9": (200, 16, 1e3, 1e-6, 9),
    "cfg1_rho1e-6": (1000, 100, 1e8, 1e-6, 11),
    "cfg1_rho1e-2": (1000, 100, 1e8, 1e-2, 12),
    "p2000_k1e4": (2000, 50, 1e4, 1e-8, 20260817),
}
probs = {}
for name, (m, n, kappa, rho, seed) in PROBLEMS.items():
    p = sq.generate_problem(m, n, kappa, rho, seed=seed)
    probs[name] = p
    meta["cases"][name] = {"m": m, "n": n, "kappa": kappa, "rho": rho, "seed": seed,
                           "sha_a": sha(p.a), "sha_b": sha(p.b), "sha_x": sha(p.x_star)}
for name in ("p300_k10_s5", "p200_k1e3_s9"):
    put(f"{name}/a", probs[name].a)
    put(f"{name}/b", probs[name].b)
    put(f"{name}/x_star", probs[name].x_star)

# 2. sketch operators and sketched matrices at every level, both transforms
for name, transform, d in (("p600_k1e2", "dct2", 120), ("p300_k10_s5", "wht", 60),
                           ("p300_k10_s5", "dct2", 60)):
    p = probs[name]
    op = sq.make_sketch(p.m, d, transform, seed=17)
    key = f"sketch/{name}/{transform}"
    put(key + "/signs", op.signs)
    put(key + "/rows", op.sampled_rows)
    for lvl in (sq.BINARY16, sq.BINARY32, sq.BINARY64):
        rounded = sq.round_to_precision(p.a, lvl)
        a_s = sq.apply_sketch(op, rounded.data)
        put(f"{key}/{lvl.name}/a_s", a_s)
        fac, err = outcome(lambda: sq.qr_in_precision(a_s, lvl))
        meta["cases"][f"{key}/{lvl.name}"] = {"qr_error": err}
        if fac is not None:
            put(f"{key}/{lvl.name}/r", fac.r)

# 3. kappa0 decisions on planted problems (auto bands)
dec = {}
for name in ("p600_k1e2", "p600_k1e6", "p600_k1e10", "p2000_k1e4", "cfg1_rho1e-6"):
    d0 = sq.decide_precision(probs[name].a)
    dec[name] = {"kappa0": d0.kappa0, "selected": d0.selected.name, "overflowed": d0.overflowed}
k_eye, o_eye = sq.estimate_log10_condition(np.eye(100))
dec["eye100"] = {"kappa0": k_eye, "overflowed": o_eye}
meta["decisions"] = dec

# 4. pipeline runs (x_hat bitwise; outcome + level + escalation)
RUNS = [
    ("p600_k1e2", "pne", "half", 4), ("p600_k1e2", "hpne", "auto", 4),
    ("p600_k1e6", "hpne", "auto", 4), ("p600_k1e10", "hpne", "auto", 4),
    ("p600_k1e6_s6", "pne", "half", 6),
    ("p600_k1e2_s3", "pne", "half", 3), ("p600_k1e2_s3", "pne", "single", 3),
    ("p600_k1e2_s3", "pne", "double", 3),
    ("cfg1_rho1e-6", "hpne", "single", 11), ("cfg1_rho1e-2", "hpne", "single", 12),
    ("p200_k1e3_s9", "pne", "double", 9),
]
runs = {}
for name, method, prec, seed in RUNS:
    p = probs[name]
    rep, err = outcome(lambda: sq.algorithm1_pipeline(p.a, p.b, method=method, precision=prec,
                                                      seed=seed, x_star=p.x_star))
    key = f"run/{name}/{method}/{prec}"
    info = {"error": err}
    if rep is not None:
        put(key + "/x_hat", rep.x_hat)
        put(key + "/r_s", rep.preconditioner.r_s)
        info.update(level=rep.preconditioner.computed_in.name,
                    escalated_from=None if rep.escalated_from is None else rep.escalated_from.name,
                    rel_error=rep.relative_error, residual_norm=rep.residual_norm,
                    relative_residual=rep.relative_residual,
                    kappa_rs=rep.preconditioner.kappa_rs, kappa_ap=rep.preconditioner.kappa_ap,
                    kappa0=None if rep.precision_decision is None else rep.precision_decision.kappa0)
    runs[key] = info
meta["runs"] = runs

# 5. unpreconditioned / two-sided solvers and the stage functions
p = probs["p300_k10_s5"]
pre = sq.build_preconditioner(p.a, seed=5)
a_p = sq.precondition_matrix(p.a, pre)
put("stage/p300_k10_s5/r_s", pre.r_s)
put("stage/p300_k10_s5/a_p", a_p)
meta["stage"] = {"kappa_rs": pre.kappa_rs, "kappa_ap": pre.kappa_ap,
                 "descriptor": pre.sketch_descriptor}
for tag, fn in (("qr", lambda: sq.solve_qr_baseline(p.a, p.b, x_star=p.x_star)),
                ("ne", lambda: sq.solve_normal(p.a, p.b, x_star=p.x_star)),
                ("sne", lambda: sq.solve_seminormal(p.a, p.b, x_star=p.x_star)),
                ("nne_ap", lambda: sq.solve_notnormal(p.a, a_p, p.b, x_star=p.x_star)),
                ("pne", lambda: sq.solve_pne(p.a, p.b, pre, x_star=p.x_star, a_p=a_p)),
                ("hpne", lambda: sq.solve_hpne(p.a, p.b, pre, x_star=p.x_star, a_p=a_p))):
    put(f"solve/p300_k10_s5/{tag}", fn().x_hat)
pn = probs["p600_k1e10"]
_, err = outcome(lambda: sq.solve_normal(pn.a, pn.b))
meta["ne_k1e10_error"] = err

# 6. known-answer vectors of the reference's own unit tests
r2 = np.array([[2.0, 1.0], [0.0, 4.0]])
put("ka/trsv", sq.triangular_solve(r2, np.array([5.0, 8.0])))
put("ka/trsv_t", sq.triangular_solve(r2, np.array([2.0, 9.0]), transposed=True))
perm = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])
put("ka/lu_perm", sq.lu_solve(perm, np.array([7.0, -2.0, 5.0])))
put("ka/round_0p1", sq.round_to_precision(np.array([0.1]), sq.BINARY16).data)
put("ka/pairwise_1001", _pairwise_sum(np.arange(1.0, 1002.0)))
dg = np.diag([1.0, 0.5, 0.25])
put("ka/hager_diag", sq.hager_one_norm_inverse_estimate(
    lambda rhs, tr: sq.triangular_solve(dg, rhs, transposed=tr), 3))
put("ka/qr_sign", sq.householder_qr(np.array([[3.0, 1.0], [4.0, 2.0]])).r)
g = sq.rng.stream(7, 3).standard_normal((9, 9))
spd = g.T @ g + np.eye(9)
put("ka/spd", spd)
put("ka/chol_x", sq.cholesky_solve(spd, np.arange(9.0)))
put("ka/lu_x", sq.lu_solve(spd + np.triu(g), np.arange(9.0)))
put("ka/jacobi_sv", sq.dense.jacobi_singular_values(g))
put("ka/rng_gauss", sq.rng.stream(123, 3).standard_normal(8))
meta["ka_mix64"] = [str(sq.rng.mix64(20260817, 3, 1)), str(sq.rng.mix64(-5, 2**62))]

np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
    json.dump(meta, fh, indent=1, default=lambda o: None if (isinstance(o, float) and math.isnan(o)) else str(o))
print("wrote", len(arrays), "arrays;", os.path.getsize(os.path.join(HERE, "golden.npz")), "bytes")
