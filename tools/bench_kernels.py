"""Per-kernel timing (CUDA events, several repetitions) at a given m x n."""
import argparse, json, math, sys, time
import torch
sys.path.insert(0, ".")
import paper_2603_16644_b200 as sq
from paper_2603_16644_b200 import dense as D, sketch as S, precision as P

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1 << 20)
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--only", default="")
args = ap.parse_args()
m, n = args.m, args.n
d = 3 * n
dev = torch.device("cuda")
g = torch.Generator(device=dev); g.manual_seed(1)
a = torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
r = torch.triu(torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)) + 8 * torch.eye(n, dtype=torch.float64, device=dev)
b = torch.randn(m, dtype=torch.float64, device=dev, generator=g)

def t(fn, reps=args.reps):
    fn(); torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); out.append(s.elapsed_time(e))
    return out

res = {}
ap_buf = torch.empty_like(a)
def want(k): return not args.only or k in args.only.split(",")
if want("syrk"):
    res["syrk"] = t(lambda: D._gram(a)); res["syrk_tflops"] = m * n * n / (min(res["syrk"]) * 1e-3) / 1e12
if want("gemm"):
    res["gemm"] = t(lambda: D._gram(a, ap_buf)); res["gemm_tflops"] = 2 * m * n * n / (min(res["gemm"]) * 1e-3) / 1e12
if want("ozaki"):
    ap_buf.normal_(generator=g)   # real data: the INT8 products draw more power than zeros
    res["oz_syrk"] = t(lambda: D._gram(a, engine="ozaki"))
    res["oz_syrk_tflops"] = m * n * n / (min(res["oz_syrk"]) * 1e-3) / 1e12
    res["oz_gemm"] = t(lambda: D._gram(a, ap_buf, engine="ozaki"))
    res["oz_gemm_tflops"] = 2 * m * n * n / (min(res["oz_gemm"]) * 1e-3) / 1e12
if want("trsm"):
    res["trsm"] = t(lambda: D._trsm(a, r, out=ap_buf)); res["trsm_tflops"] = m * n * n / (min(res["trsm"]) * 1e-3) / 1e12
    del ap_buf
    torch.cuda.empty_cache()
    res["trsm_padded"] = t(lambda: D._trsm(a, r)); res["trsm_padded_tflops"] = m * n * n / (min(res["trsm_padded"]) * 1e-3) / 1e12
    ap_buf = torch.empty_like(a)
if want("sketch"):
    op = sq.make_sketch(m, d, "dct2", seed=1); dsk = S.DeviceSketch(op)
    res["sketch_tc"] = t(lambda: S._sketch_sum(dsk, a, 16, algo="tc"))
    res["sketch_tc_tflops"] = 2 * d * m * n / (min(res["sketch_tc"]) * 1e-3) / 1e12
if want("qr"):
    op = sq.make_sketch(m, d, "dct2", seed=1); dsk = S.DeviceSketch(op)
    tot, _ = S._sketch_sum(dsk, a, 16)
    def qr16():
        a_s, _ = S._sketch_finalize(tot, op, P.BINARY16)
        P._qr_level_dev(a_s, P.BINARY16, d, n)
    res["qr16"] = t(qr16, 2)
    def qr64():
        a_s, _ = S._sketch_finalize(tot, op, P.BINARY64)
        P._qr_level_dev(a_s, P.BINARY64, d, n)
    res["qr64"] = t(qr64, 2)
if want("nxn"):
    gm = D._gram(a[: 4 * n])
    rhs = torch.randn(n, dtype=torch.float64, device=dev)
    res["chol"] = t(lambda: D._chol_solve(gm, rhs), 2)
    res["lu"] = t(lambda: D._lu_solve(gm, rhs), 2)
    res["kappa0_nxn"] = t(lambda: P._kappa0_from_gram(gm), 2)
    res["trsv"] = t(lambda: D._trsv(r, rhs), 2)
print(json.dumps({k: ([round(x, 3) for x in v] if isinstance(v, list) else round(v, 3)) for k, v in res.items()}))
