"""Box bring-up: hardware facts and the FP64 / low-precision peaks the roofline needs.

Same method as MEASURED_PEAKS.json ("how"): CUDA events, best of 10 (burst) and a
back-to-back loop for ~4 s (sustained).  Writes gpurun_out/bringup.json.
"""
import json, os, subprocess, time
import torch


def bench_mm(dtype, n=8192, reps=10, sustain_s=4.0, tf32=False):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=torch.float32).to(dtype)
    b = torch.randn(n, n, device="cuda", dtype=torch.float32).to(dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); a @ b; e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    flops = 2.0 * n ** 3
    t0 = time.time(); cnt = 0
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < sustain_s:
        for _ in range(4):
            a @ b
        cnt += 4
        torch.cuda.synchronize()
    e.record(); e.synchronize()
    sus = flops * cnt / (s.elapsed_time(e) / 1e3)
    return {"burst_tflops": flops / best / 1e12, "sustained_tflops": sus / 1e12}


def main():
    out = {}
    p = torch.cuda.get_device_properties(0)
    out["gpu"] = {"name": p.name, "sms": p.multi_processor_count, "mem_gib": p.total_memory / 2**30}
    out["host"] = {"cpu_count": os.cpu_count()}
    for cmd, key in (("lscpu", "lscpu"), ("free -g", "free"), ("nvidia-smi topo -m", "topo"),
                     ("nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.limit --format=csv", "smi"),
                     ("ncu --version", "ncu")):
        try:
            out[key] = subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout[-3000:]
        except Exception as ex:  # noqa
            out[key] = repr(ex)
    out["fp64"] = bench_mm(torch.float64)
    out["fp32_simt"] = bench_mm(torch.float32, tf32=False)
    out["tf32"] = bench_mm(torch.float32, tf32=True)
    out["fp16"] = bench_mm(torch.float16)
    # HBM copy
    x = torch.empty(2**30, dtype=torch.bfloat16, device="cuda"); y = torch.empty_like(x)
    for _ in range(3): y.copy_(x)
    best = 1e9
    for _ in range(10):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); y.copy_(x); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e) / 1e3)
    out["hbm_copy_gbs"] = 2 * x.numel() * 2 / best / 1e9
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/bringup.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("gpu", "host", "fp64", "fp32_simt", "tf32", "fp16", "hbm_copy_gbs")}))


if __name__ == "__main__":
    main()
