"""Golden hashes of the REAL reference's binary16 level QR at config-3 shapes.

Run in the build container only (needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_qr16.py [case ...]

The d = 1536 / 6144 inputs span 6 / 24 256-row chunks, so they pin the chunk-tree
decomposition of csrc/qr.cu against the reference's `_pairwise_sum`
(src/precision.py:106-115) applied over rows j..d-1 with odd tails carried, which
the single-chunk goldens of make_golden.py cannot.

Inputs are bit-reproducible without BLAS: A[:, j] = G[:, j] * s_j with
G = numpy.random.default_rng(seed).standard_normal((d, n)) and s_j a fixed
geometric column grading (elementwise IEEE products), so the GPU tests rebuild
the same bytes on the GPU box (the input's SHA-256 is stored and checked).

Each case calls the reference's own code path of qr_in_precision(a, BINARY16)
(src/precision.py:188-202): the f64 max and power-of-two scale, round_to_precision,
householder_reduce with HALF_OPS and, where `q` is set, accumulate_thin_q with
HALF_OPS.  The big case skips Q (the pipeline never forms it; build_preconditioner
discards it, src/solvers.py:196-197) to keep the run under an hour.
Writes tests/golden/qr16_golden.json (merged with existing cases).
"""
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import sketchlsq as sq  # noqa: E402
from sketchlsq.dense import accumulate_thin_q, householder_reduce  # noqa: E402
from sketchlsq.precision import BINARY16, HALF_OPS, round_to_precision  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "qr16_golden.json")

# name: (d, n, seed, log10 of the column grading span, form Q)
CASES = {
    "d1000_n333_g1": (1000, 333, 11, 1.0, True),       # odd tails at every tree level
    "d1536_n512_g1": (1536, 512, 12, 1.0, True),       # 6 chunks, Q pinned too
    "d1536_n512_g7": (1536, 512, 13, 7.0, False),      # collapses: forced-half escalation at d > 256
    "d6144_n2048_g1": (6144, 2048, 14, 1.0, False),    # config-3 shape (d = 3n), 24 chunks
}


def make_input(d, n, seed, span):
    """Shared with tests/test_gpu_qr16_golden.py (same formula, numpy only)."""
    g = np.random.default_rng(seed).standard_normal((d, n))
    s = 10.0 ** (-span * np.arange(n, dtype=np.float64) / max(n - 1, 1))
    return g * s[None, :]


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def run(name):
    d, n, seed, span, want_q = CASES[name]
    a = make_input(d, n, seed, span)
    rec = {"d": d, "n": n, "seed": seed, "span": span, "input_sha256": sha(a)}
    t0 = time.time()
    # src/precision.py:188-194
    maxabs = float(np.abs(a).max())
    _, exp = math.frexp(maxabs)
    scale = 2.0 ** -exp
    rounded = round_to_precision(a * scale, BINARY16)
    rec["scale"] = scale
    try:
        with np.errstate(over="ignore", invalid="ignore", under="ignore"):
            refl, taus, r16 = householder_reduce(rounded.data, HALF_OPS)
            q16 = accumulate_thin_q(refl, taus, d, n, ops=HALF_OPS, dtype=np.float16) if want_q else None
        if not (np.isfinite(r16).all() and (q16 is None or np.isfinite(q16).all())):
            rec["outcome"] = "Overflow"
        else:
            r = r16.astype(np.float64) / scale
            rec["outcome"] = "ok"
            rec["r_sha256"] = sha(r)
            rec["r_diag_head"] = [float(x) for x in np.diag(r)[:4]]
            rec["r_fro"] = float(np.linalg.norm(r))
            if q16 is not None:
                q = np.ascontiguousarray(q16.astype(np.float64))   # row-major f64 like QRFactors.q
                rec["q_sha256"] = sha(q)
                rec["q_fro"] = float(np.linalg.norm(q))
    except sq.SketchLsqError as ex:
        rec["outcome"] = type(ex).__name__
        rec["message"] = str(ex)
    rec["seconds"] = round(time.time() - t0, 1)
    return rec


def range_cases():
    """Small inputs outside the binary16 range (max 1e6) and in its subnormal range
    (1e-6): the reference scales on the f64 values before rounding, so both succeed.
    Full R and Q stored (tests/golden/qr16_range.json)."""
    out = {}
    for name, (d, n, seed, mag) in {"big": (40, 12, 21, 1e6), "tiny": (40, 12, 22, 1e-6),
                                    "mixed": (64, 16, 23, 3e4), "huge": (40, 12, 24, 1e300)}.items():
        a = np.random.default_rng(seed).standard_normal((d, n)) * mag
        if name == "mixed":
            a[:, ::2] *= 1e-2
        rec = {"d": d, "n": n, "seed": seed, "mag": mag, "input_sha256": sha(a)}
        try:
            f = sq.qr_in_precision(a, BINARY16)
            rec.update(outcome="ok", r=f.r.tolist(), q=f.q.tolist())
        except sq.SketchLsqError as ex:
            rec.update(outcome=type(ex).__name__)
        out[name] = rec
    with open(os.path.join(HERE, "qr16_range.json"), "w") as fh:
        json.dump(out, fh)


def main():
    if sys.argv[1:] == ["--range"]:
        range_cases()
        return
    names = sys.argv[1:] or list(CASES)
    data = json.load(open(OUT)) if os.path.exists(OUT) else {"reference": "sketchlsq " + sq.__version__, "cases": {}}
    for name in names:
        rec = run(name)
        print(name, json.dumps(rec), flush=True)
        data["cases"][name] = rec
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
