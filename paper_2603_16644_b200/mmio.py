"""Problem-archive I/O (src/mmio.py:1-37 and the archive half of src/probgen.py:126-159).

Matrix Market array files through scipy.io with 17 significant digits, so every
float64 survives a write/read round trip bitwise, exactly as the reference writes
them (archives from either package load in the other).  A Matrix Market text file of a
config-3 A (4M x 2048) would be ~170 GB of text and take hours to parse, so the
archive may also carry raw `.npy` sidecars: `save_problem(...,
sidecar=True)` writes A.npy / b.npy / xstar.npy next to (or, with `mtx=False`,
instead of) the .mtx files and lists them in meta.json under "sidecar"; `load_problem`
memory-maps the sidecars when present (the solvers stream a host A to the GPU in
chunks), else reads the .mtx files.  meta.json keeps the reference's keys and
format_version, so the reference's load_problem still reads an archive with .mtx files.
"""

from __future__ import annotations

import json
import os

import numpy as np

FORMAT_VERSION = 1          # src/probgen.py:22
SIDECAR_AUTO_ELEMENTS = 1 << 24   # save_problem(sidecar=None): .npy sidecars from 16M entries of A


def write_matrix(path, a):
    """src/mmio.py:13-20: dense matrix or vector (as one column) to a Matrix Market array file."""
    from scipy.io import mmwrite
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a[:, None]
    if a.ndim != 2:
        raise ValueError(f"expected 1-D or 2-D data, got ndim={a.ndim}")
    mmwrite(str(path), a, precision=17)


def read_matrix(path):
    """src/mmio.py:23-28: a Matrix Market file as a dense 2-D float64 array."""
    from scipy.io import mmread
    data = mmread(str(path))
    if hasattr(data, "toarray"):
        data = data.toarray()
    return np.asarray(data, dtype=np.float64)


def read_vector(path):
    """src/mmio.py:31-37: a single-row or single-column file as a 1-D array."""
    data = read_matrix(path)
    if data.ndim == 2 and data.shape[1] == 1:
        return data[:, 0].copy()
    if data.ndim == 2 and data.shape[0] == 1:
        return data[0, :].copy()
    raise ValueError(f"expected a single row or column, got shape {data.shape}")


_FILES = (("a", "A"), ("b", "b"), ("x_star", "xstar"))


def save_problem(problem, directory, *, sidecar=None, mtx=True):
    """src/probgen.py:126-143: A.mtx, b.mtx, xstar.mtx + meta.json; plus .npy sidecars
    when `sidecar` (default: A has >= 16M entries).  `mtx=False` skips the text files
    (then only this package's load_problem reads the archive)."""
    a = np.asarray(problem.a)
    if sidecar is None:
        sidecar = a.size >= SIDECAR_AUTO_ELEMENTS
    if not (mtx or sidecar):
        raise ValueError("save_problem needs mtx=True or sidecar=True")
    os.makedirs(directory, exist_ok=True)
    for field, stem in _FILES:
        value = getattr(problem, field)
        if mtx:
            write_matrix(os.path.join(directory, f"{stem}.mtx"), value)
        if sidecar:
            np.save(os.path.join(directory, f"{stem}.npy"), np.ascontiguousarray(value, dtype=np.float64))
    meta = {"format_version": FORMAT_VERSION, "m": int(a.shape[0]), "n": int(a.shape[1]),
            "kappa": problem.kappa, "rho": problem.rho, "seed": problem.seed}
    if sidecar:
        meta["sidecar"] = [f"{stem}.npy" for _, stem in _FILES]
    with open(os.path.join(directory, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=2)
        fh.write("\n")


def load_problem(directory, *, mmap=True):
    """src/probgen.py:146-159: the archived problem, bitwise; .npy sidecars (memory-
    mapped unless mmap=False) take precedence over the .mtx files."""
    from .probgen import LeastSquaresProblem
    with open(os.path.join(directory, "meta.json")) as fh:
        meta = json.load(fh)
    version = meta.get("format_version")
    if version != FORMAT_VERSION:
        raise ValueError(f"unsupported archive format_version {version!r}")
    arrays = {}
    for field, stem in _FILES:
        npy = os.path.join(directory, f"{stem}.npy")
        if os.path.exists(npy):
            v = np.load(npy, mmap_mode="r" if mmap else None)
            if v.dtype != np.float64:
                raise ValueError(f"{stem}.npy holds {v.dtype}, expected float64")
        elif field == "a":
            v = read_matrix(os.path.join(directory, "A.mtx"))
        else:
            v = read_vector(os.path.join(directory, f"{stem}.mtx"))
        arrays[field] = v
    if arrays["a"].shape != (meta["m"], meta["n"]):
        raise ValueError(f"A shape {arrays['a'].shape} disagrees with meta {meta['m']}x{meta['n']}")
    if arrays["b"].ndim != 1 or arrays["x_star"].ndim != 1:
        raise ValueError("b and xstar must be vectors")
    return LeastSquaresProblem(a=arrays["a"], b=arrays["b"], x_star=arrays["x_star"], rho=float(meta["rho"]),
                               kappa=float(meta["kappa"]), seed=int(meta["seed"]))
