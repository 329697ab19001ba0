"""The shared-memory-resident dataflow LU (lu_smem_kernel, the default for n <= 2048)
against the one-barrier-per-step lu_perm_kernel (SK_LU_KERNEL=perm): both are
op-for-op the reference's partial-pivoting LU (src/dense.py:245-286), so the
factors, the pivot sequence and x agree bit for bit, ties and failures included.
The kernel choice is read once per process, so each arm runs in its own process."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2603_16644_b200 as sq
from oracle import restatement as R
out = {}
for n, kind in ((2048, "gauss"), (2048, "ties"), (1500, "gauss"), (64, "ties"), (2048, "singular"),
                (1, "gauss"), (2, "ties"), (31, "gauss"), (32, "ties"), (33, "gauss"), (100, "gauss"),
                (160, "ties"), (161, "gauss"), (120, "singular")):
    g = R.philox(n, 11)
    if kind == "ties":
        a = g.integers(-2, 3, size=(n, n)).astype(np.float64)   # many equal pivot magnitudes
    else:
        a = g.standard_normal((n, n))
    if kind == "singular":
        a[:, min(700, n - 1)] = a[:, 3] * 2.0
    rhs = g.standard_normal(n)
    key = f"{n}_{kind}"
    try:
        out[key] = sq.lu_solve(a, rhs)
    except sq.NumericallySingular as ex:
        out[key] = np.array([float("nan")])
        out[key + "_err"] = np.frombuffer(str(ex).encode(), dtype=np.uint8)
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, tag, env_extra):
    env = dict(os.environ)
    env.pop("SK_LU_KERNEL", None)
    env.update(env_extra)
    path = str(tmp_path / f"{tag}.npz")
    subprocess.run([sys.executable, "-c", SCRIPT, ROOT, path], check=True, env=env, cwd=ROOT, timeout=600)
    return dict(np.load(path))


@pytest.mark.gpu
def test_smem_lu_bitwise_equals_perm_lu(tmp_path):
    """default (one-CTA lu_small_kernel for n <= 160, lu_smem_kernel above) vs
    SK_LU_KERNEL=smem (the dataflow kernel at every n <= 2048) vs SK_LU_KERNEL=perm."""
    smem = _run(tmp_path, "default", {})
    flow = _run(tmp_path, "smem", {"SK_LU_KERNEL": "smem"})
    perm = _run(tmp_path, "perm", {"SK_LU_KERNEL": "perm"})
    assert sorted(smem) == sorted(perm) == sorted(flow)
    for k in smem:
        assert np.array_equal(smem[k], perm[k], equal_nan=True), k
        assert np.array_equal(flow[k], perm[k], equal_nan=True), k
    assert "120_singular_err" in smem
    assert "2048_singular_err" in smem                       # NumericallySingular, same column and value
    assert np.isfinite(smem["2048_gauss"]).all() and np.isfinite(smem["2048_ties"]).all()
