"""The level QR with shared-memory-resident columns (householder_flow_kernel<T, true>,
the default whenever a CTA's columns fit) against the global-memory flow kernel
(SK_QR_SMEM=0): the same chunk trees and rounding points, so R agrees bit for bit at
every level -- also when only a CTA's later columns fit shared memory (binary32 / binary64
at 6144 x 2048) --
every level, including the binary16 collapse that drives the escalation
(src/precision.py:153-202, src/solvers.py:255-279).  The choice is read once per
process, so each arm runs in its own process."""
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
cases = [(6144, 2048, "binary16", 1.0), (3000, 1000, "binary32", 1.0), (1200, 400, "binary64", 1.0),
         (6144, 2048, "binary32", 1.0), (6144, 2048, "binary64", 1.0),   # partly shared-memory resident
         (700, 300, "binary16", 1.0), (600, 40, "binary16", 1e-6), (1001, 333, "binary16", 1.0)]   # odd d: no half2 pairs
for d, n, lev, spread in cases:
    g = R.philox(d + n, 5)
    a = g.standard_normal((d, n)) * np.logspace(0, np.log10(spread), n)   # spread < 1: graded columns
    key = f"{d}x{n}_{lev}_{spread:g}"
    try:
        out[key] = sq.qr_in_precision(a, getattr(sq, lev.upper())).r
    except sq.RankDeficient as ex:
        out[key] = np.array([float("nan")])
        out[key + "_err"] = np.frombuffer(str(ex).encode(), dtype=np.uint8)
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, tag, env_extra):
    env = dict(os.environ)
    env.pop("SK_QR_SMEM", None)
    env.update(env_extra)
    path = str(tmp_path / f"{tag}.npz")
    subprocess.run([sys.executable, "-c", SCRIPT, ROOT, path], check=True, env=env, cwd=ROOT, timeout=600)
    return dict(np.load(path))


@pytest.mark.gpu
def test_smem_qr_bitwise_equals_global_qr(tmp_path):
    smem = _run(tmp_path, "smem", {})
    glob = _run(tmp_path, "global", {"SK_QR_SMEM": "0"})
    assert sorted(smem) == sorted(glob)
    for k in smem:
        assert np.array_equal(smem[k], glob[k], equal_nan=True), k
    assert np.isfinite(smem["6144x2048_binary16_1"]).all()
