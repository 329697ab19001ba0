"""Re-measure the two roofline denominators MEASURED_PEAKS.json does not carry, with the
SM clock and throttle reasons sampled during each measurement (bench.py's ClockSampler):
FP64 DGEMM (torch.matmul float64, cuBLAS: the TRSM leaf's and the DMMA Gram's peak) and
INT8 GEMM with int32 accumulation (torch._int_mm, cuBLASLt: the Ozaki engine's peak),
each as best-of-10 (burst) and back to back for 4 s (sustained).

    python tools/peaks_with_clocks.py > profiles/r2_peaks_with_clocks.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def measure(fn, flops, reps=10, sustain_s=4.0):
    import torch
    from bench import ClockSampler
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    torch.cuda.synchronize()
    t = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    count = 0
    while time.perf_counter() - t < sustain_s:
        fn()
        count += 1
        if count % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    sus = e0.elapsed_time(e1) * 1e-3 / count
    return {"burst": flops / best / 1e12, "sustained": flops / sus / 1e12, "clocks_sustained": clocks.stop()}


def main():
    import torch
    out = {"gpu": torch.cuda.get_device_name(0)}
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    out["fp64_dgemm_tflops"] = measure(lambda: torch.matmul(a, b), 2.0 * n ** 3)
    del a, b
    m, k, nn = 2048, 131072, 2048
    x = torch.randint(-127, 128, (m, k), dtype=torch.int8, device="cuda")
    y = torch.randint(-127, 128, (k, nn), dtype=torch.int8, device="cuda")
    out["int8_gemm_tops"] = measure(lambda: torch._int_mm(x, y), 2.0 * m * k * nn)
    out["shapes"] = {"fp64": f"{n}^3", "int8": f"{m} x {k} x {nn} (the Gram's K-long shape)"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
