"""Host staging-copy bandwidth (pageable numpy -> pinned), the bound of the pageable e2e
path: torch copy_ at several intra-op thread counts, and numpy copyto split over N Python
threads (GIL released in the copy)."""
import json, os, sys, time, threading
import numpy as np
import torch

nbytes = 256 << 20
n = nbytes // 8
src_np = np.random.default_rng(0).standard_normal(n * 8).reshape(8, n)   # 2 GiB pageable, touched
dst = torch.empty(n, dtype=torch.float64, pin_memory=True)
dst_np = dst.numpy()
out = {"cpu_count": os.cpu_count(), "torch_threads_default": torch.get_num_threads()}

def bw(fn, reps=8):
    fn(0)
    t = time.perf_counter()
    for i in range(reps):
        fn(i % 8)
    return nbytes * reps / (time.perf_counter() - t) / 1e9

for th in (1, 4, 8, 16, 32):
    torch.set_num_threads(th)
    out[f"torch_copy_threads_{th}_GBs"] = bw(lambda i: dst.copy_(torch.from_numpy(src_np[i])))

def np_threads(k):
    def fn(i):
        s = src_np[i]
        parts = np.array_split(np.arange(n), k)
        ts = [threading.Thread(target=np.copyto, args=(dst_np[p[0]:p[-1] + 1], s[p[0]:p[-1] + 1])) for p in parts]
        for t in ts: t.start()
        for t in ts: t.join()
    return fn

for k in (1, 4, 8, 16):
    out[f"numpy_copyto_{k}_threads_GBs"] = bw(np_threads(k))
print(json.dumps(out))
