"""Config 5 at FULL size (1,048,576 x 1024, d = 3072) over the whole
kappa x rho grid, GPU against the row-chunked hybrid CPU oracle (oracle/hybrid.py) for
every method the survey lists: pne and hpne (precision auto), sne, nne with B = A_p and
with B = A.

Per kappa one planted problem A = Q1 R (probgen.generate_problem_device; A depends only
on the seed), b_rho = A x* + rho e for every rho (e the unit residual direction, e ⟂
range(A)).  The oracle side computes everything that depends on A alone once per kappa
(kappa0 and the level decision, the sketch, the level QR with its escalation, A_p per
row chunk, the Grams A_p^T A_p / A_p^T A / A^T A, R of A by LAPACK for sne) and the
right-hand sides A_p^T b_rho, A^T b_rho per rho; the n x n solves are the reference's
(restatement).  Gate per (kappa, rho, method): the same outcome class, level and
escalation, relative error <= max(10 x oracle, 1e-14).  One JSON line per point.

    python tools/config5_parity.py [--m 1048576] [--n 1024] [--kappas ...] [--rhos ...]
"""
import argparse
import json
import math
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

KAPPAS = "1e2,1e4,1e6,1e8,1e10,1e12,1e14"
RHOS = "1e-14,1e-12,1e-10,1e-8,1e-6,1e-4,1e-2,1e-1"


def outcome(fn):
    try:
        return "ok", fn()
    except Exception as ex:  # noqa: BLE001 (compared by class name)
        return type(ex).__name__, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1 << 20)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--kappas", default=KAPPAS)
    ap.add_argument("--rhos", default=RHOS)
    ap.add_argument("--seed", type=int, default=20261019)
    args = ap.parse_args()
    import numpy as np
    import scipy.linalg
    import torch

    import paper_2603_16644_b200 as sq
    from oracle import hybrid as H
    from oracle import restatement as R
    from paper_2603_16644_b200.probgen import generate_problem_device

    m, n = args.m, args.n
    rhos = [float(x) for x in args.rhos.split(",")]
    for kappa in [float(k) for k in args.kappas.split(",")]:
        t_k = time.perf_counter()
        a, b1, xs = generate_problem_device(m, n, kappa, 1.0, args.seed)
        _, b0, _ = generate_problem_device(m, n, kappa, 0.0, args.seed)
        torch.cuda.synchronize()
        e = b1 - b0
        del b1
        a_h = a.cpu().numpy()
        b0_h, e_h, xs_h = b0.cpu().numpy(), e.cpu().numpy(), xs.cpu().numpy()
        seed = args.seed + 1

        # ---------------- oracle: everything that depends on A alone
        tm = {}
        t = time.perf_counter()
        k0, over = H.kappa0(a_h)
        level = R.choose_level(k0, over)
        tm["kappa0"] = time.perf_counter() - t
        failed, pre_err, r_s = None, None, None
        while True:
            try:
                t = time.perf_counter()
                a_s, _ = H.sketch(a_h, level, 3.0, "dct2", seed)
                r_s = H.level_r(a_s, level)
                if (np.diagonal(r_s) == 0).any():
                    raise R.RankDeficient("zero diagonal")
                tm["sketch_qr"] = tm.get("sketch_qr", 0.0) + time.perf_counter() - t
                break
            except R.RankDeficient as ex:
                wider = R.WIDER.get(level)
                if failed is not None or wider is None:
                    pre_err = type(ex).__name__
                    break
                failed, level = level, wider
            except R.Overflow as ex:
                pre_err = type(ex).__name__
                break
        t = time.perf_counter()
        g_pne = g_hpne = None
        c_p = np.zeros((n, 2))                        # A_p^T [b0 e]
        if r_s is not None:
            g_pne, g_hpne = np.zeros((n, n)), np.zeros((n, n))
            for r0 in range(0, m, H.CHUNK):
                ac = a_h[r0:r0 + H.CHUNK]
                apc = scipy.linalg.solve_triangular(r_s, ac.T, trans="T", lower=False, check_finite=False).T
                g_pne += apc.T @ apc
                g_hpne += apc.T @ ac
                c_p += apc.T @ np.stack([b0_h[r0:r0 + H.CHUNK], e_h[r0:r0 + H.CHUNK]], axis=1)
        g_a = H._gram_chunked(a_h)
        c_a = a_h.T @ np.stack([b0_h, e_h], axis=1)
        tm["grams"] = time.perf_counter() - t
        t = time.perf_counter()
        r_a = scipy.linalg.qr(a_h, mode="r", overwrite_a=False, check_finite=False)[0][:n]   # LAPACK dgeqrf
        tm["lapack_qr"] = time.perf_counter() - t

        def ref_solve(method, rho):
            if method in ("pne", "hpne") and pre_err is not None:
                raise getattr(R, pre_err)("preconditioner")
            if method == "pne":
                rhs = c_p[:, 0] + rho * c_p[:, 1]
                try:
                    y = R.spd_solve(g_pne, rhs)
                except R.NotPositiveDefinite:
                    y = R.lu_pivoted_solve(g_pne, rhs)
                return R.tri_solve(r_s, y)
            if method in ("hpne", "nne_ap"):
                return R.lu_pivoted_solve(g_hpne, c_p[:, 0] + rho * c_p[:, 1])
            if method == "nne_a":
                return R.lu_pivoted_solve(g_a, c_a[:, 0] + rho * c_a[:, 1])
            if method == "sne":
                rhs = c_a[:, 0] + rho * c_a[:, 1]
                return R.tri_solve(r_a, R.tri_solve(r_a, rhs, transposed=True))
            raise ValueError(method)

        # ---------------- GPU: the package's public API
        dec = sq.decide_precision(a)
        gpu_pre = outcome(lambda: sq.prepare_preconditioner(a, 3.0, "dct2", dec.selected, seed,
                                                            diagnostics=False))
        for rho in rhos:
            b = b0 + rho * e
            b_h = b0_h + rho * e_h
            rec = {"m": m, "n": n, "kappa": kappa, "rho": rho,
                   "oracle_decision": {"kappa0": k0, "overflowed": over, "level": level, "escalated_from": failed,
                                       "preconditioner": pre_err or "ok"},
                   "gpu_decision": {"kappa0": dec.kappa0, "overflowed": dec.overflowed,
                                    "level": dec.selected.name}, "methods": {}}
            gpu_runs = {
                "pne": lambda: sq.algorithm1_pipeline(a, b, "pne", "auto", 3.0, "dct2", seed, xs, diagnostics=False),
                "hpne": lambda: sq.algorithm1_pipeline(a, b, "hpne", "auto", 3.0, "dct2", seed, xs,
                                                       diagnostics=False),
                "sne": lambda: sq.solve_seminormal(a, b, xs),
                "nne_ap": lambda: sq.solve_notnormal(a, gpu_pre[1][1], b, xs),
                "nne_a": lambda: sq.solve_notnormal(a, a, b, xs),
            }
            ok_all = True
            for meth, run in gpu_runs.items():
                if meth == "nne_ap" and gpu_pre[0] != "ok":
                    g_out, g_rep = gpu_pre[0], None
                else:
                    torch.cuda.synchronize()
                    t = time.perf_counter()
                    g_out, g_rep = outcome(run)
                    torch.cuda.synchronize()
                    g_ms = (time.perf_counter() - t) * 1e3
                r_out, x_ref = outcome(lambda: ref_solve(meth, rho))
                r_err = (float(np.linalg.norm(x_ref - xs_h) / np.linalg.norm(xs_h))
                         if x_ref is not None and np.isfinite(x_ref).all() else None)
                g_err = g_rep.relative_error if g_rep is not None else None
                entry = {"gpu_outcome": g_out, "oracle_outcome": r_out, "gpu_rel_error": g_err,
                         "oracle_rel_error": r_err}
                if g_rep is not None:
                    entry["gpu_ms"] = g_ms
                    if g_rep.preconditioner is not None:
                        entry["gpu_level"] = g_rep.preconditioner.computed_in.name
                        entry["gpu_escalated_from"] = g_rep.escalated_from.name if g_rep.escalated_from else None
                ok = g_out == r_out
                if ok and g_err is not None and r_err is not None:
                    ok = g_err <= max(10 * r_err, 1e-14) or not math.isfinite(r_err)
                if meth in ("pne", "hpne") and g_rep is not None:
                    ok = ok and entry.get("gpu_level") == level and entry.get("gpu_escalated_from") == failed
                entry["gate_ok"] = bool(ok)
                ok_all = ok_all and ok
                rec["methods"][meth] = entry
            rec["gate_ok"] = ok_all
            rec["oracle_seconds_per_kappa"] = tm
            print(json.dumps(rec), flush=True)
        del a, b0, e, a_h
        torch.cuda.empty_cache()
        print(json.dumps({"kappa": kappa, "seconds": time.perf_counter() - t_k}), file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
