"""Config 2 (100000 x 1000) through the numpy-in / numpy-out API, warm, call by call."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2603_16644_b200 as sq
from oracle import restatement as R
from oracle.problems import planted_problem_lapack

p = planted_problem_lapack(100000, 1000, 1e10, 1e-6, R.mix64(20261018, 2))


def t(label, fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        s = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        out.append(round((time.perf_counter() - s) * 1e3, 1))
    print(json.dumps({label: out}))
    return r


pre = t("build_preconditioner", lambda: sq.build_preconditioner(p.a, 3.0, "dct2", sq.BINARY32, 0, diagnostics=False))
ap = t("precondition_matrix", lambda: sq.precondition_matrix(p.a, pre, diagnostics=False))
t("solve_pne(numpy a_p)", lambda: sq.solve_pne(p.a, p.b, pre, x_star=p.x_star, a_p=ap, diagnostics=False))
t("solve_hpne(numpy a_p)", lambda: sq.solve_hpne(p.a, p.b, pre, x_star=p.x_star, a_p=ap, diagnostics=False))
at = torch.from_numpy(p.a).cuda()
bt = torch.from_numpy(p.b).cuda()
pre_t = sq.build_preconditioner(at, 3.0, "dct2", sq.BINARY32, 0, diagnostics=False)
apt = sq.precondition_matrix(at, pre_t, diagnostics=False)
t("solve_pne(device)", lambda: sq.solve_pne(at, bt, pre_t, x_star=p.x_star, a_p=apt, diagnostics=False))
t("solve_hpne(device)", lambda: sq.solve_hpne(at, bt, pre_t, x_star=p.x_star, a_p=apt, diagnostics=False))
t("pipeline hpne single (numpy)", lambda: sq.algorithm1_pipeline(p.a, p.b, "hpne", "single", diagnostics=False))
t("pipeline hpne single (device)", lambda: sq.algorithm1_pipeline(at, bt, "hpne", "single", diagnostics=False))
