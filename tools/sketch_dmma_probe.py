"""Time the dense DMMA sketch at config-2 shape (100000 x 1000, d = 3000, binary32 level)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_16644_b200.sketch import _make_sketch_dev, _sketch_sum
m, n = int(sys.argv[1]), int(sys.argv[2])
lev = int(sys.argv[3]) if len(sys.argv) > 3 else 32
d = 3 * n
a = torch.randn(m, n, dtype=torch.float64, device="cuda")
op, dsk = _make_sketch_dev(m, d, "dct2", 1)
for _ in range(2):
    _sketch_sum(dsk, a, lev, algo="dmma")
torch.cuda.synchronize()
ms = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); _sketch_sum(dsk, a, lev, algo="dmma"); e1.record(); e1.synchronize()
    ms.append(e0.elapsed_time(e1))
print(json.dumps({"m": m, "n": n, "d": d, "level": lev, "ms": min(ms), "tflops": 2 * d * m * n / min(ms) / 1e9}))
