"""Sketch engines at config-3 size: CUDA-event time per call (sk_sketch_partial_ex),
the fraction of the one-read-of-A HBM floor, and agreement between engines.

    python tools/bench_sketch.py [--m 4194304] [--n 2048] [--levels 16,32,64] [--algos tc,fft]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4 * 1024 * 1024)
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--levels", default="16,32,64")
    ap.add_argument("--algos", default="tc,fft")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--row-offset", type=int, default=0)
    args = ap.parse_args()
    import torch
    from paper_2603_16644_b200.sketch import _make_sketch_dev, _sketch_sum
    m, n = args.m, args.n
    d = 3 * n
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    op, dsk = _make_sketch_dev(m + args.row_offset, d, "dct2", 1)
    out = {}
    ref = None
    for lv in [int(x) for x in args.levels.split(",")]:
        for algo in args.algos.split(","):
            if algo == "tc" and lv != 16:
                continue
            try:
                tot, _ = _sketch_sum(dsk, a, lv, row_offset=args.row_offset, algo=algo)
                torch.cuda.synchronize()
                ts = []
                for _ in range(args.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    tot, _ = _sketch_sum(dsk, a, lv, row_offset=args.row_offset, algo=algo)
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
            except Exception as ex:  # noqa: BLE001
                out[f"{algo}{lv}"] = {"error": repr(ex)}
                continue
            ms = min(ts)
            rec = {"ms": ms, "ms_all": ts, "hbm_floor_frac": 8.0 * m * n / (ms * 1e-3) / 6451.8e9}
            if lv == 64 and algo == "fft":
                ref = tot.clone()
            out[f"{algo}{lv}"] = rec
            if ref is not None and lv != 64:
                rec["max_rel_vs_fft64"] = ((tot - ref).abs().max() / ref.abs().max()).item()
    print(json.dumps({"m": m, "n": n, "d": d, "row_offset": args.row_offset, "results": out}))


if __name__ == "__main__":
    main()
