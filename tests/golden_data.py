"""Loader for the committed reference fixtures (tests/golden/)."""
import hashlib
import json
import os

import numpy as np

from oracle import problems

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ARR = np.load(os.path.join(HERE, "golden.npz"))
META = json.load(open(os.path.join(HERE, "golden_meta.json")))
_CACHE = {}


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def problem(name):
    """Regenerate a golden problem with the oracle generator (pinned by hash)."""
    if name not in _CACHE:
        c = META["cases"][name]
        _CACHE[name] = problems.planted_problem(c["m"], c["n"], c["kappa"], c["rho"], c["seed"])
    return _CACHE[name]
