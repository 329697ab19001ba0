"""CPU oracle for the sketch-preconditioned normal-equations hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2603_16644_b200`) imports this package.  It may be imported by
`tests/`, by `__graft_entry__.smoke()` (as the checker) and by `bench.py`'s
`cpu_baseline` / `--impl reference` legs (as the timed CPU baseline).

`restatement` re-states, in plain numpy/scipy, the algorithm of the reference
package `sketchlsq` 0.1.0 (arXiv 2603.16644, `/root/reference/pkg/src/sketchlsq`)
operation for operation, so that on the same inputs it returns bit-identical
results to the reference in the same environment.  Each function cites the
reference file:line it follows.  `problems` re-states the Algorithm-2 problem
generator (`probgen.py`) so the GPU box, which has no `/root/reference`, can
build the same planted problems from seeds.

Parity is PINNED: `tests/golden/make_golden.py` imports the real reference in
the build container and stores its outputs under `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this restatement against them bitwise.
"""

from . import restatement, problems  # noqa: F401
