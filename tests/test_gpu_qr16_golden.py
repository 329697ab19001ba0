"""Level QR pinned bitwise to the REAL reference at config-3 shapes.

Goldens from tests/golden/make_golden_qr16.py (the reference's own
qr_in_precision code path, src/precision.py:153-202, run in the build container):
SHA-256 of the binary16 R (and Q where formed) for d x n inputs that span 4-24
256-row chunks, so the chunk-tree decomposition of csrc/qr.cu is compared with the
reference's `_pairwise_sum` over rows j..d-1 (src/precision.py:106-115); the
forced-half collapse column at d > 256; and full R / Q for inputs outside the
binary16 range (the prescale is taken on the f64 values before rounding,
src/precision.py:188-194).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2603_16644_b200 as sq

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLD = json.load(open(os.path.join(HERE, "qr16_golden.json")))["cases"]
RANGE = json.load(open(os.path.join(HERE, "qr16_range.json")))


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def make_input(d, n, seed, span):
    """Same formula as make_golden_qr16.make_input (elementwise, BLAS-free)."""
    g = np.random.default_rng(seed).standard_normal((d, n))
    s = 10.0 ** (-span * np.arange(n, dtype=np.float64) / max(n - 1, 1))
    return g * s[None, :]


@pytest.mark.parametrize("name", sorted(GOLD))
def test_binary16_qr_bitwise_reference(name):
    c = GOLD[name]
    a = make_input(c["d"], c["n"], c["seed"], c["span"])
    assert sha(a) == c["input_sha256"], "input regeneration differs from the golden run"
    if c["outcome"] != "ok":
        with pytest.raises(getattr(sq, c["outcome"])) as ei:
            sq.qr_in_precision(a, sq.BINARY16)
        # the reference names the collapsing column ("reflector 220 norm underflowed ...")
        col = [int(t) for t in c["message"].split() if t.isdigit()]
        assert col and str(col[0]) in str(ei.value), (c["message"], str(ei.value))
        return
    f = sq.qr_in_precision(a, sq.BINARY16)
    assert float(np.diag(f.r)[0]) == c["r_diag_head"][0]
    assert sha(f.r) == c["r_sha256"], "binary16 R differs from the reference's bits"
    if "q_sha256" in c:
        assert sha(np.ascontiguousarray(f.q)) == c["q_sha256"], "binary16 Q differs from the reference's bits"


@pytest.mark.parametrize("name", sorted(RANGE))
def test_binary16_qr_outside_fp16_range(name):
    c = RANGE[name]
    a = np.random.default_rng(c["seed"]).standard_normal((c["d"], c["n"])) * c["mag"]
    if name == "mixed":
        a[:, ::2] *= 1e-2
    assert sha(a) == c["input_sha256"]
    if c["outcome"] != "ok":
        with pytest.raises(getattr(sq, c["outcome"])):
            sq.qr_in_precision(a, sq.BINARY16)
        return
    f = sq.qr_in_precision(a, sq.BINARY16)
    np.testing.assert_array_equal(f.r, np.array(c["r"]))
    np.testing.assert_array_equal(f.q, np.array(c["q"]))


def test_pipeline_qr_matches_public_qr_at_6144():
    """The pipeline's level QR (sk_qr_r on an already-demoted fp16 sketch) and the
    public qr_in_precision give the same bits when the input is fp16-exact and
    already prescaled."""
    import torch
    from paper_2603_16644_b200.precision import _qr_level_dev
    c = GOLD["d6144_n2048_g1"]
    a = make_input(c["d"], c["n"], c["seed"], c["span"])
    scaled = (a * c["scale"]).astype(np.float16)
    work = torch.from_numpy(np.asfortranarray(scaled).T.copy()).cuda()   # column-major d x n
    r_pipe = _qr_level_dev(work, sq.BINARY16, c["d"], c["n"]).cpu().numpy() / c["scale"]
    assert sha(r_pipe) == c["r_sha256"]


@pytest.mark.parametrize("level", ["BINARY32", "BINARY64"])
def test_level_q_orthonormal_and_reconstructs(level):
    a = make_input(1000, 333, 11, 3.0)
    f = sq.qr_in_precision(a, getattr(sq, level))
    u = 2.0 ** -23 if level == "BINARY32" else 2.0 ** -52
    n = a.shape[1]
    assert np.abs(f.q.T @ f.q - np.eye(n)).max() <= 100 * n * u
    assert np.abs(f.q @ f.r - a).max() <= 100 * n * u * np.abs(a).max()
    assert np.all(np.tril(f.r, -1) == 0)


def test_householder_reduce_reflectors_and_accumulate_q():
    """householder_reduce returns the reference's (reflectors, taus, R) layout;
    accumulate_thin_q from them reproduces householder_qr's Q; the sign convention
    R00 = -5 for [3, 4] (tests/test_dense.py:41-47)."""
    from oracle import restatement as R
    a = make_input(700, 90, 5, 2.0)
    refl, taus, r = sq.householder_reduce(a)
    assert len(refl) == 90 and len(taus) == 90
    assert [v.shape[0] for v in refl[:3]] == [700, 699, 698]
    for j in (0, 17, 89):
        assert taus[j] == pytest.approx(2.0 / float(refl[j] @ refl[j]), rel=1e-14)
    ro_refl, ro_taus, ro_r = R.householder_steps(a)
    np.testing.assert_allclose(r, ro_r, rtol=1e-12, atol=1e-12 * np.abs(ro_r).max())
    np.testing.assert_allclose(refl[5], ro_refl[5], rtol=1e-10, atol=1e-12)
    q = sq.accumulate_thin_q(refl, taus, 700, 90)
    f = sq.householder_qr(a)
    np.testing.assert_array_equal(q, f.q)
    np.testing.assert_array_equal(r, f.r)
    _, _, r2 = sq.householder_reduce(np.array([[3.0], [4.0]]))
    assert r2[0, 0] == -5.0
