"""Micro-benchmark + check of sk_gram_f64 (SYRK and GEMM-TN) against cuBLAS."""
import ctypes as C, sys, time, json
import torch
sys.path.insert(0, ".")
from paper_2603_16644_b200 import _lib

L = _lib.lib()
dev = torch.device("cuda")

def ev_time(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return min(ts)

res = {}
for (m, n) in [(1000, 40), (5000, 333), (65536, 512), (1 << 20, 2048)]:
    x = torch.randn(m, n, device=dev, dtype=torch.float64)
    y = torch.randn(m, n, device=dev, dtype=torch.float64)
    g = torch.empty(n, n, device=dev, dtype=torch.float64)
    wsb = L.sk_gram_workspace(m, n)
    ws = torch.empty(wsb // 8 + 1, device=dev, dtype=torch.float64)
    s = torch.cuda.current_stream().cuda_stream
    def run_syrk():
        rc = L.sk_gram_f64(x.data_ptr(), n, x.data_ptr(), n, m, n, g.data_ptr(), n, 0, ws.data_ptr(), wsb, s)
        assert rc == 0, _lib.last_error()
    def run_gemm():
        rc = L.sk_gram_f64(x.data_ptr(), n, y.data_ptr(), n, m, n, g.data_ptr(), n, 0, ws.data_ptr(), wsb, s)
        assert rc == 0, _lib.last_error()
    run_syrk(); torch.cuda.synchronize()
    ref = x.T @ x
    e1 = ((g - ref).abs().max() / ref.abs().max()).item()
    sym = (g - g.T).abs().max().item()
    run_gemm(); torch.cuda.synchronize()
    ref2 = x.T @ y
    e2 = ((g - ref2).abs().max() / ref2.abs().max()).item()
    t_s = ev_time(run_syrk); t_g = ev_time(run_gemm)
    t_cub = ev_time(lambda: torch.matmul(x.T, y))
    fl = 2.0 * m * n * n
    r = dict(m=m, n=n, err_syrk=e1, sym=sym, err_gemm=e2, syrk_ms=t_s, gemm_ms=t_g, cublas_gemm_ms=t_cub,
             syrk_tf=fl / 2 / t_s / 1e9, gemm_tf=fl / t_g / 1e9, cublas_tf=fl / t_cub / 1e9)
    print(json.dumps(r)); res[f"{m}x{n}"] = r
    del x, y, g, ws; torch.cuda.empty_cache()
