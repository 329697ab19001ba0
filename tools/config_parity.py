"""Full-size parity + timing for the non-headline measurement configurations (SURVEY
§8(d)), GPU against the oracle port on this box's host cores:

  config 1  1000 x 100, kappa 1e8, HPNE "single", rho grid       (parity, CPU vs GPU time)
  config 2  100000 x 1000, kappa 1e10, rho 1e-6, PNE and HPNE sharing one fixed
            binary32 preconditioner                             (parity, CPU vs GPU time)
  config 5  1M x 1024, kappa x rho grid, pne / hpne auto       (GPU vs planted x*; the
            oracle on two grid points: it needs minutes per point on the host)

Writes one JSON document to stdout (profiles/r1_config_parity.json)."""
import json, math, os, sys, time
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2603_16644_b200 as sq
from oracle import restatement as R
from oracle.problems import planted_problem, planted_problem_lapack
from paper_2603_16644_b200.probgen import generate_problem_device


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t) * 1e3


def outcome(fn):
    try:
        return "ok", fn()
    except Exception as e:  # noqa: BLE001 (compared by class name)
        return type(e).__name__, None


out = {"host_cores": os.cpu_count()}

# ---- config 1
c1 = []
for rho in (1e-16, 1e-12, 1e-8, 1e-4, 1.0):
    p = planted_problem(1000, 100, 1e8, rho, R.mix64(20261018, 1, int(-math.log10(rho)) if rho < 1 else 0))
    sq.algorithm1_pipeline(p.a, p.b, "hpne", "single", 3.0, "dct2", 0, p.x_star, diagnostics=False)
    g, g_ms = timed(lambda: sq.algorithm1_pipeline(p.a, p.b, "hpne", "single", 3.0, "dct2", 0, p.x_star,
                                                   diagnostics=False))
    t = time.perf_counter()
    r = R.pipeline(p.a, p.b, "hpne", "single", 3.0, "dct2", 0, p.x_star, diagnostics=False)
    c_ms = (time.perf_counter() - t) * 1e3
    c1.append({"rho": rho, "gpu_ms": g_ms, "cpu_ms": c_ms, "gpu_rel_error": g.relative_error,
               "oracle_rel_error": r.relative_error, "level": g.preconditioner.computed_in.name,
               "within_gate": g.relative_error <= max(10 * r.relative_error, 1e-14)})
out["config1"] = c1

# ---- config 2
p = planted_problem_lapack(100000, 1000, 1e10, 1e-6, R.mix64(20261018, 2))
t = time.perf_counter()
pre_r = R.build_pre(p.a, 3.0, "dct2", "binary32", 0, diagnostics=False)
ap_r = R.precondition(p.a, pre_r, diagnostics=False)
cpu_pre_ms = (time.perf_counter() - t) * 1e3
c2 = {"cpu_preconditioner_ms": cpu_pre_ms}
(pre, gpu_pre_ms) = timed(lambda: sq.build_preconditioner(p.a, 3.0, "dct2", sq.BINARY32, 0, diagnostics=False))
ap, gpu_ap_ms = timed(lambda: sq.precondition_matrix(p.a, pre, diagnostics=False))
c2["gpu_preconditioner_ms"] = gpu_pre_ms + gpu_ap_ms
for meth, fr, fo in (("pne", R.solve_pne, sq.solve_pne), ("hpne", R.solve_hpne, sq.solve_hpne)):
    t = time.perf_counter()
    ref = outcome(lambda: fr(p.a, p.b, pre_r, x_star=p.x_star, a_p=ap_r))
    cpu_ms = (time.perf_counter() - t) * 1e3
    ours, gpu_ms = timed(lambda: outcome(lambda: fo(p.a, p.b, pre, x_star=p.x_star, a_p=ap, diagnostics=False)))
    c2[meth] = {"cpu_ms": cpu_ms, "gpu_ms": gpu_ms, "outcome": ours[0], "oracle_outcome": ref[0],
                "gpu_rel_error": ours[1].relative_error if ours[1] else None,
                "oracle_rel_error": ref[1].relative_error if ref[1] else None}
    if ours[1] and ref[1]:
        c2[meth]["within_gate"] = ours[1].relative_error <= max(10 * ref[1].relative_error, 1e-14)
out["config2"] = c2

# ---- config 5 (GPU grid against x*; the oracle on two points)
m, n = 1 << 20, 1024
c5 = []
for kappa in (1e2, 1e4, 1e6, 1e8, 1e10, 1e12, 1e14):
    for rho in (1e-14, 1e-10, 1e-6, 1e-2):
        a, b, xs = generate_problem_device(m, n, kappa, rho, R.mix64(20261018, 5, int(math.log10(kappa)),
                                                                   int(-math.log10(rho))), torch.device("cuda"))
        row = {"kappa": kappa, "rho": rho}
        for meth in ("pne", "hpne"):
            o, ms = timed(lambda: outcome(lambda: sq.algorithm1_pipeline(a, b, meth, "auto", 3.0, "dct2", 0, xs,
                                                                         diagnostics=False)))
            row[meth] = {"ms": ms, "outcome": o[0], "rel_error": o[1].relative_error if o[1] else None,
                         "level": o[1].preconditioner.computed_in.name if o[1] else None}
        qr = outcome(lambda: sq.solve_qr_baseline(a, b, x_star=xs))
        row["qr_baseline_rel_error"] = qr[1].relative_error if qr[1] else qr[0]
        if (kappa, rho) in ((1e6, 1e-6), (1e10, 1e-6)):
            ah, bh, xh = a.cpu().numpy(), b.cpu().numpy(), xs.cpu().numpy()
            t = time.perf_counter()
            ref = outcome(lambda: R.pipeline(ah, bh, "hpne", "auto", 3.0, "dct2", 0, xh, diagnostics=False))
            row["oracle_hpne"] = {"cpu_ms": (time.perf_counter() - t) * 1e3, "outcome": ref[0],
                                  "rel_error": ref[1].relative_error if ref[1] else None,
                                  "level": ref[1].pre.level if ref[1] else None}
            del ah
        c5.append(row)
        del a, b, xs
        torch.cuda.empty_cache()
out["config5"] = c5
print(json.dumps(out))
