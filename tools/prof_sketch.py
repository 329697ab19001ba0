"""Small driver for ncu captures of the sketch kernels (1M x 2048)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2603_16644_b200 as sq
from paper_2603_16644_b200 import sketch as S
m, n, d = 1 << 20, 2048, 6144
a = torch.randn(m, n, dtype=torch.float64, device="cuda")
op = sq.make_sketch(m, d, "dct2", seed=1)
dsk = S.DeviceSketch(op)
for _ in range(2):
    S._sketch_sum(dsk, a, 16, algo="tc")
    S._sketch_sum(dsk, a, 64, algo="fft")
torch.cuda.synchronize()
print("ok")
