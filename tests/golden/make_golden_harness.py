"""Golden fixtures for the harness / CLI / bounds row, made by running
the REAL reference (`sketchlsq` 0.1.0) in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_harness.py

Writes
  harness_golden.json   bound formulas (src/bounds.py:55-156) on fixed inputs, incl.
                        the PoleAtOne / MissingField / ValueError cases; rho_grid;
                        sample_size_lower_bound; one reference run_sweep (all five
                        methods, double and auto) and one run_benchmark, rows without
                        wall_ms / timings
  archive_ref/          a small problem archive written by the reference's gen command
                        (Matrix Market + meta.json), for the bitwise load test
"""
import json
import os
import shutil
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import sketchlsq as sq  # noqa: E402
from sketchlsq import bounds as B  # noqa: E402
from sketchlsq.cli import main as ref_main  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
out = {"reference": "sketchlsq " + sq.__version__}


def outcome(fn):
    try:
        return {"value": fn()}
    except Exception as ex:  # noqa: BLE001
        return {"raises": type(ex).__name__}


# 1. bound formulas
full = dict(kappa_a=1e6, kappa_rs=3.5, kappa_ap=1.7, kappa_apta=2.2e5, nu_pne=0.9, nu_hpne=1.3, u1=2.0 ** -11,
            u2=2.0 ** -52, eps_a=2.0 ** -52, eps_b=2.0 ** -24, eps_p=2.0 ** -52, eps_s=2.0 ** -11,
            res_ratio_a=3e-7, res_ratio_ap=4e-9)
cases = {"full": full,
         "pole": dict(full, kappa_rs=2.0 ** 11),
         "missing_rs": {k: v for k, v in full.items() if k != "kappa_rs"},
         "missing_eps_b": {k: v for k, v in full.items() if k != "eps_b"},
         "large": dict(full, kappa_a=1e14, kappa_rs=1e7, kappa_ap=40.0, u1=2.0 ** -24, res_ratio_a=1e-2)}
bounds = {}
for name, kw in cases.items():
    bi = B.BoundInputs(**kw)
    bounds[name] = {"inputs": kw, "results": {
        "bound_ls": outcome(lambda: B.bound_ls(bi)),
        "bound_ne_family": outcome(lambda: B.bound_ne_family(bi)),
        "bound_ne_family_seminormal": outcome(lambda: B.bound_ne_family(bi, "seminormal")),
        "bound_ne_family_bad": outcome(lambda: B.bound_ne_family(bi, "other")),
        "bound_pne_old": outcome(lambda: B.bound_pne(bi, "old")),
        "bound_pne_new": outcome(lambda: B.bound_pne(bi, "new")),
        "bound_pne_bad": outcome(lambda: B.bound_pne(bi, "x")),
        "bound_hpne_old": outcome(lambda: B.bound_hpne(bi, "old")),
        "bound_hpne_new": outcome(lambda: B.bound_hpne(bi, "new")),
        "bound_notnormal": outcome(lambda: B.bound_notnormal(bi, 12.5, 1.1)),
        "eta1": outcome(lambda: B.eta1(bi.kappa_rs, bi.u1) if bi.kappa_rs is not None else None),
    }}
out["bounds"] = bounds

# 2. rho_grid, sample_size_lower_bound
out["rho_grid"] = {"1e-16,1,33": sq.rho_grid(1e-16, 1.0, 33).tolist(), "1e-8,1,5": sq.rho_grid(1e-8, 1.0, 5).tolist(),
                   "1e-3,1e-3,1": sq.rho_grid(1e-3, 1e-3, 1).tolist()}
out["sample_size"] = {f"{m},{n},{mu},{eps},{dl}": sq.sample_size_lower_bound(sq.EmbeddingParams(m, n, mu, eps, dl))
                      for (m, n, mu, eps, dl) in ((1000, 100, 0.2, 0.5, 0.01), (4194304, 2048, 0.001, 0.9, 1e-3))}

# 3. sweeps (rows without wall_ms)
SWEEPS = {
    "double": dict(m=120, n=10, kappa=1e3, rho_grid=sq.rho_grid(1e-10, 1e-2, 3),
                   methods=("qr", "ne", "pne", "hpne", "sne"), precision="double", trials_per_point=2, seed=17),
    "auto": dict(m=300, n=20, kappa=1e2, rho_grid=sq.rho_grid(1e-8, 1e-4, 2), methods=("qr", "pne", "hpne"),
                 precision="auto", trials_per_point=1, seed=5),
    "failure": dict(m=200, n=12, kappa=1e9, rho_grid=sq.rho_grid(1e-8, 1e-8, 1), methods=("qr", "ne"),
                    precision="double", trials_per_point=1, seed=17),
}
sweeps = {}
for name, kw in SWEEPS.items():
    cfg = dict(kw)
    cfg_json = dict(kw, rho_grid=list(map(float, kw["rho_grid"])), methods=list(kw["methods"]))
    rows = sq.run_sweep(sq.SweepConfig(**cfg))
    sweeps[name] = {"config": cfg_json, "rows": [{k: v for k, v in r.items() if k != "wall_ms"} for r in rows]}
out["sweeps"] = sweeps

bench = sq.run_benchmark(m=160, n_list=(8, 12), kappa=1e3, rho=1e-6, trials=1, seed=3)
out["benchmark"] = {"args": dict(m=160, n_list=[8, 12], kappa=1e3, rho=1e-6, trials=1, seed=3),
                    "rows": [{k: r[k] for k in ("method", "m", "n", "kappa", "trials", "rel_error")} for r in bench]}

with open(os.path.join(HERE, "harness_golden.json"), "w") as fh:
    json.dump(out, fh, indent=1, default=float)
    fh.write("\n")

# 4. a reference-written archive
arch = os.path.join(HERE, "archive_ref")
shutil.rmtree(arch, ignore_errors=True)
assert ref_main(["gen", "--m", "40", "--n", "6", "--kappa", "1e3", "--rho", "1e-6", "--seed", "5", "--out", arch]) == 0
p = sq.load_problem(arch)
with open(os.path.join(HERE, "archive_ref_sha.json"), "w") as fh:
    import hashlib
    json.dump({k: hashlib.sha256(np.ascontiguousarray(getattr(p, k)).tobytes()).hexdigest()
               for k in ("a", "b", "x_star")}, fh, indent=1)
    fh.write("\n")
print("wrote harness_golden.json, archive_ref/")
