"""TRSM timing variance probe: per-rep CUDA-event time next to the SM clock and
power sampled by nvidia-smi every 50 ms during that rep."""
import subprocess, sys, threading, time, json
import torch
sys.path.insert(0, ".")
from paper_2603_16644_b200 import dense as D
m, n = 1 << 22, 2048
g = torch.Generator(device="cuda"); g.manual_seed(1)
a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
r = torch.triu(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)) + 8 * torch.eye(n, dtype=torch.float64, device="cuda")
out = torch.empty_like(a)
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
lines = []
th = threading.Thread(target=lambda: [lines.append((time.time(), l.strip())) for l in proc.stdout], daemon=True)
th.start()
D._trsm(a, r, out=out); torch.cuda.synchronize()
res = []
for i in range(8):
    t0 = time.time()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); D._trsm(a, r, out=out); e.record(); e.synchronize()
    t1 = time.time()
    samp = [l for (t, l) in lines if t0 <= t <= t1]
    clk = [float(x.split(",")[1]) for x in samp if len(x.split(",")) > 2]
    pw = [float(x.split(",")[2]) for x in samp if len(x.split(",")) > 2]
    res.append({"ms": round(s.elapsed_time(e), 1), "sm_mhz_min": min(clk) if clk else None,
                "sm_mhz_med": sorted(clk)[len(clk) // 2] if clk else None, "power_max": max(pw) if pw else None,
                "reasons": sorted(set(x.split(",")[3].strip() for x in samp if len(x.split(",")) > 3))})
proc.terminate()
for x in res: print(json.dumps(x))
