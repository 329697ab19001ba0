"""Where the config-1 solve's time goes (device-resident A, b): wall per solve, the
GPU busy time of its kernels (torch.profiler / CUPTI, all kernels of the process), the
host-side Python profile (cProfile, top functions by cumulative time) and the number of
blocking host reads.

    python tools/latency_breakdown.py [--method hpne] [--precision single]
"""
import argparse
import cProfile
import io
import json
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1000)
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--method", default="hpne")
    ap.add_argument("--precision", default="single")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--kappa", type=float, default=1e8)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2603_16644_b200 as sq
    from oracle.problems import planted_problem
    if args.m * args.n <= 4_000_000:
        p = planted_problem(args.m, args.n, args.kappa, 1e-6, 11)
    else:                                     # large: the device generator, copied to the host
        from paper_2603_16644_b200.probgen import generate_problem_device
        from types import SimpleNamespace
        a_d, b_d, x_d = generate_problem_device(args.m, args.n, args.kappa, 1e-6, 11)
        p = SimpleNamespace(a=a_d.cpu().numpy(), b=b_d.cpu().numpy(), x_star=x_d.cpu().numpy())
    a, b = torch.from_numpy(p.a).cuda(), torch.from_numpy(p.b).cuda()

    def solve():
        return sq.algorithm1_pipeline(a, b, method=args.method, precision=args.precision, seed=1,
                                      diagnostics=False)
    for _ in range(5):
        solve()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(args.reps):
        solve()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / args.reps * 1e3
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(args.reps):
            solve()
        torch.cuda.synchronize()
    kern, syncs, memcpy = {}, 0, 0
    gpu_us = 0.0
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            kern.setdefault(e.name, [0, 0.0])
            kern[e.name][0] += 1
            kern[e.name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
            gpu_us += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        elif "Synchronize" in e.name:
            syncs += 1
        elif "Memcpy" in e.name and "Async" not in e.name:
            memcpy += 1
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(args.reps):
        solve()
    torch.cuda.synchronize()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
    out = {"m": args.m, "n": args.n, "kappa": args.kappa, "method": args.method, "precision": args.precision,
           "wall_ms_per_solve": wall, "gpu_kernel_ms_per_solve": gpu_us / 1e3 / args.reps,
           "sync_calls_per_solve": syncs / args.reps, "blocking_memcpy_per_solve": memcpy / args.reps,
           "kernels": {k: {"per_solve": v[0] / args.reps, "us_per_solve": v[1] / args.reps}
                       for k, v in sorted(kern.items(), key=lambda kv: -kv[1][1])}}
    # the same solve as one CUDA graph (PipelinePlan: deferred verdicts, one host read)
    from paper_2603_16644_b200.graph import PipelinePlan
    plan = PipelinePlan(args.m, args.n, method=args.method, precision=args.precision, seed=1)
    ref = solve()
    for kind, (aa, bb) in {"device": (a, b), "numpy": (p.a, p.b)}.items():
        for _ in range(5):
            rep = plan.solve(aa, bb)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(args.reps):
            rep = plan.solve(aa, bb)
        torch.cuda.synchronize()
        out["graph_" + kind] = {"ms_per_solve": (time.perf_counter() - t) / args.reps * 1e3,
                                "x_bitwise_equal_eager": bool((rep.x_hat == ref.x_hat).all())}
    t = time.perf_counter()
    for _ in range(args.reps):
        sq.algorithm1_pipeline(p.a, p.b, method=args.method, precision=args.precision, seed=1, diagnostics=False)
    torch.cuda.synchronize()
    out["eager_numpy_ms_per_solve"] = (time.perf_counter() - t) / args.reps * 1e3
    with profile(activities=[ProfilerActivity.CUDA]) as prof2:
        for _ in range(args.reps):
            plan.solve(a, b)
        torch.cuda.synchronize()
    gk = [e for e in prof2.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    out["graph_kernels_per_solve"] = len(gk) / args.reps
    out["graph_gpu_ms_per_solve"] = sum(getattr(e, "device_time_total", 0) for e in gk) / 1e3 / args.reps
    print(json.dumps(out, indent=1))
    print(s.getvalue(), file=sys.stderr)


if __name__ == "__main__":
    main()
