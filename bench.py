"""Benchmark: Algorithm-1 solve time at 4M x 2048 (BASELINE.json config 3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one full `algorithm1_pipeline(A, b, method, precision="auto")`
solve (kappa0 estimate, sketch, level QR, A_p = A R^-1, Gram, n x n solve,
residual report) on device-resident synthetic data of prescribed kappa(A) and
residual (the GPU Algorithm-2 generator, probgen.py).  `value` is milliseconds
per solve (lower is better) timed with CUDA events between barriers, max over
ranks.  `e2e` is the same solve through the public API from pinned HOST
buffers, the host->device copy of A and b and the device->host read of x_hat
inside the timed region.  A (68.7 GB) is far larger than L2, so no flush is
needed between steps.

Multi-GPU (torchrun): rows are sharded, each rank holds m rows (weak scaling:
m_total = N * m); partial Gram / sketch results are summed with NCCL
all-reduce (distributed.py).

`--impl reference` times the reference algorithm on the host CPU (the oracle
port in oracle/, all host threads) on a bounded sample of the same workload and
reports it in the same unit, extrapolated stage by stage to the full size.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
# A, A_p and the sketch operand are 64/64/16 GiB at config 3: avoid caching-allocator
# fragmentation between the generator's and the solver's large blocks.
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

METRIC = "PNE/HPNE solve time at 4M×2048 (1–8 GPUs); % of roofline; rel. error"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--m", type=int, default=None,
                   help="total rows (default: config 3, 4M, at N = 1; config 4, 16M row-sharded, at N > 1)")
    p.add_argument("--n", type=int, default=2048)
    p.add_argument("--kappa", type=float, default=10.0)
    p.add_argument("--rho", type=float, default=1e-6)
    p.add_argument("--method", default="hpne", choices=["pne", "hpne"])
    p.add_argument("--precision", default="auto")
    p.add_argument("--seed", type=int, default=20261018)
    p.add_argument("--e2e-steps", type=int, default=1)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-e2e-pageable", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-config1", action="store_true", help="skip the config-1 latency report")
    p.add_argument("--cpu-rows", type=int, default=8192, help="row-slice height (full n) for the CPU legs")
    return p.parse_args()


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sms.append(float(parts[0]))
                maxs.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": max(maxs) if maxs else None,
                "reasons": sorted(reasons), "samples": len(sms)}


# -------------------------------------------------------------- roofline ---
def fp64_peak():
    """Measured cuBLAS DGEMM peak (TFLOP/s) from profiles/, else the spec estimate."""
    path = os.path.join(HERE, "profiles", "fp64_peak.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["fp64_tflops"]), d.get("source", path)
    except Exception:  # noqa: BLE001
        return 37.2, "spec estimate 148 SM x 64 FMA/clk x 2 x 1.965 GHz (not measured)"


def hbm_peak():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def _peak_file(name, key, fallback, why):
    try:
        with open(os.path.join(HERE, "profiles", name)) as fh:
            d = json.load(fh)
        return float(d[key]), d.get("source", name)
    except Exception:  # noqa: BLE001
        return fallback, why


def int8_peak():
    return _peak_file("int8_peak.json", "int8_tops", 3100.0, "fallback: cuBLASLt INT8 on B200 (not measured)")


def fp16_peak():
    return _peak_file("fp64_peak.json", "fp16_tflops_burst", 1546.0, "fallback: cuBLAS fp16 on B200 (not measured)")


OZ_P = (255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193, 191)   # csrc/ozaki.cu pm()
OZ_TRSM_MODULI = 15     # csrc/ozaki.cu trsm_rec: |C'| < 2^113 at h = 1024, t = 51


def gram_moduli(m):
    """csrc/ozaki.cu gram_moduli: fewest leading moduli with t >= 68 - log2 m (cap 51)."""
    import math
    L = math.log2(max(m, 1))
    tmin = min(51, math.ceil(68.0 - L))
    lg = 0.0
    for k, p in enumerate(OZ_P):
        lg += math.log2(p)
        t = min(51, math.floor((lg - 1.0 - L - 0.01) / 2.0))
        if t >= tmin:
            return k + 1
    return len(OZ_P)


def oz_residue_bytes(nm):
    return 8 + nm          # per element and operand: 8 read + nm residue bytes written


TRSM_LEAF = 1024        # csrc/ozaki.cu: blocked TRSM leaves (SK_TRSM_OZ_BASE default)


def trsm_blocks(n, base=TRSM_LEAF):
    """The blocked TRSM's recursion (csrc/ozaki.cu trsm_split / trsm_rec): leaf widths
    and (h, w) of every INT8 update."""
    if n <= base:
        return [n], []
    h = min((n // 2 + 255) // 256 * 256, 2048)
    l1, u1 = trsm_blocks(h, base)
    l2, u2 = trsm_blocks(n - h, base)
    return l1 + l2, u1 + [(h, n - h)] + u2


def trsm_roofline(m, n, blocked):
    """TRSM stage roofline (s): FP64 DMMA leaves m nl^2 / DMMA peak; each update as 16
    INT8 products 2 m h w / INT8 peak plus its HBM passes (A_p[:, :h] read + 16 residue
    planes written: 24 B per element; 16 product planes written and read, A read, A_p
    written: 48 B per element of m x w)."""
    p64, p8, hbm = fp64_peak()[0] * 1e12, int8_peak()[0] * 1e12, hbm_peak()[0] * 1e9
    if not blocked:
        return float(m) * n * n / p64
    leaves, ups = trsm_blocks(n)
    t = sum(float(m) * nl * nl for nl in leaves) / p64
    for h, w in ups:
        t += 2.0 * OZ_TRSM_MODULI * m * h * w / p8 + ((8.0 + OZ_TRSM_MODULI) * m * h +
                                                             (2 * OZ_TRSM_MODULI + 16.0) * m * w) / hbm
    return t


def engine_roofline(m, n, d, method, auto, ozaki, trsm_blocked=False):
    """Roofline of the implemented solve, engine by engine (ms):
    TRSM on FP64 DMMA (blocked: DMMA leaves + INT8 updates, trsm_roofline); the kappa0
    SYRK and the PNE/HPNE Gram on the INT8 tensor cores (16 exact modular products,
    symmetric half for SYRKs) plus their residue and column-scan HBM passes; the
    binary16 sketch on the fp16 tensor cores (or one read of A if that is slower); the
    residual pass on HBM."""
    p64, p8, p16, hbm = fp64_peak()[0] * 1e12, int8_peak()[0] * 1e12, fp16_peak()[0] * 1e12, hbm_peak()[0] * 1e9
    el = float(m) * n
    t = {"trsm": trsm_roofline(m, n, trsm_blocked), "report": 8 * el / hbm,
         "sketch": max(2.0 * d * el / p16, 10 * el / hbm)}

    def gram(syrk):
        if not ozaki:
            return (1.0 if syrk else 2.0) * el * n / p64
        nm = gram_moduli(m)
        ops = 2.0 * nm * el * n * (0.5 if syrk else 1.0)
        return ops / p8 + (1 if syrk else 2) * (oz_residue_bytes(nm) + 8) * el / hbm
    if auto:
        t["kappa0"] = gram(True)
    t["gram"] = gram(method != "hpne")
    return t


def time_trsm_leaf(a, m, n, nl, reps=3):
    """One DMMA leaf launch of the blocked TRSM (A[:, :nl] at pitch n -> A_p scratch at
    pitch n, as the solve issues it), CUDA events on the current stream, ms per launch."""
    import ctypes as C
    import torch
    from paper_2603_16644_b200 import _lib, release_scratch
    from paper_2603_16644_b200.device import call, stream_handle
    release_scratch()
    out = torch.empty_like(a)
    g = torch.Generator(device=a.device)
    g.manual_seed(3)
    r = torch.triu(torch.randn(n, n, dtype=torch.float64, device=a.device, generator=g)) + \
        8 * torch.eye(n, dtype=torch.float64, device=a.device)
    st = _lib.SkStatus()

    def leaf():
        call("sk_trsm_right_upper_f64", a.data_ptr(), n, m, nl, r.data_ptr(), n, out.data_ptr(), n,
             C.byref(st), stream_handle())
    leaf()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        leaf()
    e1.record()
    torch.cuda.synchronize()
    del out
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / reps


def ncu_traffic(kernel_key):
    try:
        with open(os.path.join(HERE, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(kernel_key)
    except Exception:  # noqa: BLE001
        return None


def stage_work(stage, m, n, d, method, level):
    """Algorithmic work per stage: (flops, bytes, bound)."""
    if stage == "kappa0":
        return float(m) * n * n, 8.0 * m * n, "tensor"          # SYRK: m n^2 flops
    if stage == "trsm":
        return float(m) * n * n, 16.0 * m * n, "tensor"
    if stage == "gram":
        f = 2.0 * m * n * n if method == "hpne" else float(m) * n * n
        return f, 16.0 * m * n if method == "hpne" else 8.0 * m * n, "tensor"
    if stage == "sketch":
        return 2.0 * d * m * n, 8.0 * m * n, "hbm"              # floor: one read of A
    if stage == "report":
        return 2.0 * m * n, 8.0 * m * n, "hbm"
    if stage == "trsm_gram":      # chunked A_p: TRSM and Gram interleaved per row chunk
        f = float(m) * n * n + (2.0 * m * n * n if method == "hpne" else float(m) * n * n)
        return f, 24.0 * m * n, "tensor"
    return None


# ------------------------------------------------------------- CPU legs ----
class CpuReference:
    """The reference algorithm on the host CPU (the oracle port, oracle/), measured
    stage by stage on the FULL column count n and scaled only in m:

    m-linear stages, timed every step on a row slice of m_s x n (m_s = --cpu-rows; the
    slice's working set is far beyond the last-level cache, so the per-row cost is the
    full-size regime) and multiplied by M / m_s (the sketch's DCT by M log M / (m_s log m_s)):
      kappa0 Gram  a.T @ a                                   src/precision.py:230
      sketch       demotion, signs, pocketfft DCT-II, rows   src/sketch.py:138-169
      A_p          the reference's column-substitution TRSM  src/dense.py:231-236
      Gram + rhs   a_p.T @ a (HPNE) / a_p.T @ a_p, a_p.T @ b  src/solvers.py:230-231, :251
      residual     a @ x - b                                 src/solvers.py:99-117
    m-independent stages, timed once per run at their FULL size:
      kappa0 n x n (Cholesky + Hager)        src/precision.py:231-251
      level QR of the d x n sketch           src/precision.py:153-202 (binary16: the C
                                             restatement of the emulated Householder,
                                             bitwise the reference's R; the reference's own
                                             numpy emulation takes ~1 h at 6144 x 2048)
      n x n LU (HPNE) / Cholesky + TRSV (PNE) src/dense.py:245-342
    The solve time reported is the sum: the reference's time per solve at M x n, modelled
    from measured full-n pieces (the shipped path cannot hold a 68.7 GB A)."""

    def __init__(self, args):
        import numpy as np
        self.args = args
        self.M, self.n = total_rows(args), args.n
        self.ms = min(args.cpu_rows, self.M)
        self.d = int(math.ceil(3.0 * self.n))
        rng = np.random.default_rng(12345)
        cols = 10.0 ** (-math.log10(max(args.kappa, 1.0)) * np.arange(self.n) / max(self.n - 1, 1))
        self.a = rng.standard_normal((self.ms, self.n)) * cols[None, :]   # a full-n slice, kappa ~ args.kappa
        self.b = rng.standard_normal(self.ms)
        self.level = {"auto": "binary16" if args.kappa <= 25 else ("binary32" if args.kappa < 5e5 else "binary64"),
                      }.get(args.precision, None) or __import__("oracle.restatement", fromlist=["x"]).canonical_level(
                          args.precision)
        self.fixed = None
        self.spent = 0.0

    def _t(self, fn):
        t = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t
        self.spent += dt
        return out, dt

    def fixed_stages(self):
        """m-independent stages at full size (once)."""
        import numpy as np
        from oracle import hybrid
        from oracle import restatement as R
        if self.fixed is not None:
            return self.fixed
        f = {}
        g = self.a.T @ self.a
        _, f["kappa0_nxn"] = self._t(lambda: R.kappa0_from_gram(g))
        # the d x n sketch of a d-row block (the level QR's input shape and value range)
        blk = np.resize(self.a, (self.d, self.n)) if self.ms < self.d else self.a[: self.d]
        _, f["level_qr"] = self._t(lambda: hybrid.level_r(R.demote(blk, self.level)[0].astype(np.float64), self.level))
        if self.args.method == "hpne":
            _, f["nxn"] = self._t(lambda: R.lu_pivoted_solve(g, self.a.T @ self.b))
        else:
            def pne_nxn():
                y = R.spd_solve(g, self.a.T @ self.b)
                return R.tri_solve(np.triu(g) + np.eye(self.n), y)
            _, f["nxn"] = self._t(pne_nxn)
        self.fixed = f
        return f

    def step(self):
        """One timed sample of the m-linear stages; returns the modelled ms per solve."""
        import numpy as np
        from oracle import restatement as R
        a, b, M, ms = self.a, self.b, self.M, self.ms
        t = {}
        _, t["kappa0_gram"] = self._t(lambda: a.T @ a)
        data, _ = R.demote(a, self.level)
        op = R.draw_sketch(ms, self.d, "dct2", 1)
        _, t["sketch"] = self._t(lambda: R.sketch_apply(op, data))
        r = np.triu(np.random.default_rng(3).standard_normal((self.n, self.n))) + self.n * np.eye(self.n)
        ap, t["trsm"] = self._t(lambda: np.ascontiguousarray(R.tri_solve(r, a.T, transposed=True).T))
        if self.args.method == "hpne":
            _, t["gram"] = self._t(lambda: (ap.T @ a, ap.T @ b))
        else:
            _, t["gram"] = self._t(lambda: (ap.T @ ap, ap.T @ b))
        x = np.ones(self.n)
        _, t["report"] = self._t(lambda: np.linalg.norm(a @ x - b))
        scale = {k: M / ms for k in t}
        scale["sketch"] = (M * math.log2(M)) / (ms * math.log2(ms))
        full = {k: v * scale[k] for k, v in t.items()}
        full.update(self.fixed_stages())
        self.last = {"sample_s": t, "full_s": full}
        return sum(full.values()) * 1e3

    def describe(self):
        return (f"oracle port of sketchlsq algorithm1_pipeline ({self.args.method}, level {self.level}, "
                f"diagnostics off) on the host: m-linear stages timed on a {self.ms} x {self.n} row slice "
                f"(full n) and scaled by M/m_s = {self.M / self.ms:g} (sketch by M log M / m_s log m_s), "
                f"m-independent stages (kappa0 n x n, level QR {self.d} x {self.n}, n x n solve) timed once at "
                f"full size; numpy/OpenBLAS + pocketfft, {cpu_cores()} threads")


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads") for i in threadpool_info() if i.get("internal_api") == "openblas"]
        if th:
            return int(th[0])
    except Exception:  # noqa: BLE001
        pass
    return os.cpu_count()


def run_reference(args, rank, world):
    if rank != 0:
        return
    ref = CpuReference(args)
    vals = []
    wall0 = time.perf_counter()
    for i in range(args.warmup + args.steps):
        v = ref.step()
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
            "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (full-n row slice)", "config": workload_config(args),
            "cpu_baseline": {"value": value, "unit": "ms", "cores": cpu_cores(), "kind": "port",
                             "sample": ref.describe()},
            "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "stages_s": ref.last["full_s"], "sample_stages_s": ref.last["sample_s"],
            "run_seconds": time.perf_counter() - wall0, "measured_seconds": ref.spent,
            "note": ("value = modelled reference time per solve at the full size (sum of the stages); "
                     "run_seconds is the wall time this arm actually spent")}
    print(json.dumps(line), flush=True)


CONFIG3_M = 4 * 1024 * 1024
CONFIG4_M = 16 * 1024 * 1024


def total_rows(args):
    return args.m if args.m else (CONFIG3_M if args.gpus == 1 else CONFIG4_M)


def workload_config(args):
    m = total_rows(args)
    name = "config 3" if (args.gpus == 1 and m == CONFIG3_M) else ("config 4" if m == CONFIG4_M else "custom")
    return {"workload": (f"{name}: A {m:,} x {args.n} fp64, {args.gpus} GPU(s) x {m // args.gpus:,} rows "
                         f"(one global planted problem, contiguous row shards), kappa(A)={args.kappa:g}, "
                         f"residual rho={args.rho:g}, {args.method.upper()}, precision={args.precision}, "
                         f"d=3n DCT-II sketch"),
            "m_total": m, "m_per_gpu": m // args.gpus, "n": args.n, "kappa": args.kappa, "rho": args.rho,
            "method": args.method, "precision": args.precision, "d_factor": 3.0, "transform": "dct2",
            "l2": "inputs larger than L2 (A is 8 m n bytes >> 126 MB): no flush needed",
            "parallelism": f"row-shard x{args.gpus} (NCCL all-reduce of the kappa0 Gram, sketch, Gram + rhs)"}


# --------------------------------------------------------------- our arm ----
def run_ours(args, rank, world):
    import numpy as np
    import torch
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200 import _lib
    from paper_2603_16644_b200.probgen import generate_problem_device

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    m_total, n = total_rows(args), args.n
    if m_total % world:
        raise SystemExit(f"rows {m_total} not divisible by {world} ranks")
    m = m_total // world
    d = int(math.ceil(3.0 * n))
    # one global planted problem: the same R and x* on every rank, Q1_g and e_g per rank
    a, b, x_star = generate_problem_device(m, n, args.kappa, args.rho, args.seed, dev, rank=rank, world=world)
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    def solve(A, B, method=None):
        method = method or args.method
        if dist is not None:
            from paper_2603_16644_b200.distributed import algorithm1_pipeline_sharded
            return algorithm1_pipeline_sharded(A, B, method=method, precision=args.precision, seed=1,
                                               x_star=x_star, diagnostics=False, stage_timing=True)
        return sq.algorithm1_pipeline(A, B, method=method, precision=args.precision, seed=1, x_star=x_star,
                                      diagnostics=False, stage_timing=True)

    lib = _lib.lib()
    for _ in range(args.warmup):
        rep = solve(a, b)
    torch.cuda.synchronize()
    barrier()
    clocks = ClockSampler(dev.index)
    clocks.start()
    l0 = lib.sk_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    e0.record()
    reps = [solve(a, b) for _ in range(args.steps)]
    e1.record()
    torch.cuda.synchronize()
    barrier()
    launches = lib.sk_launch_count() - l0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # the metric names both solvers: time the other one on the same A, b (after the
    # headline's timed region, same protocol: warm-up, then args.steps timed solves)
    other = "pne" if args.method == "hpne" else "hpne"
    solve(a, b, other)
    torch.cuda.synchronize()
    barrier()
    o0 = torch.cuda.Event(enable_timing=True)
    o1 = torch.cuda.Event(enable_timing=True)
    o0.record()
    oreps = [solve(a, b, other) for _ in range(args.steps)]
    o1.record()
    torch.cuda.synchronize()
    barrier()
    oms = o0.elapsed_time(o1) / args.steps
    if dist is not None:
        t = torch.tensor([oms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        oms = float(t.item())
    other_line = {"method": other, "ms_per_step": oms, "rel_error": oreps[-1].relative_error,
                  "selected_level": oreps[-1].preconditioner.computed_in.name}
    del oreps
    rep = reps[-1]
    stages = {}
    for r in reps:
        for k, v in r.stage_ms.items():
            stages[k] = stages.get(k, 0.0) + v / len(reps)
    level = rep.preconditioner.computed_in.name
    summary = {"selected_level": level, "kappa0": rep_kappa0(rep),
               "escalated_from": rep.escalated_from.name if rep.escalated_from else None,
               "rel_error": rep.relative_error, "relative_residual": rep.relative_residual}

    # roofline of the dominant stage (CUDA events around the stage, same stream)
    from paper_2603_16644_b200.dense import _gram_engine, _trsm_engine
    ozaki = _gram_engine(m, n, False, None) == "ozaki"
    if ozaki and "check" in stages and args.precision == "auto":
        stages["kappa0"] = stages.get("kappa0", 0.0) + stages.pop("check")   # the kappa0 SYRK runs in "check"
    trsm_blocked = _trsm_engine(m, n, False, None) == "ozaki"
    dom = max((k for k in stages if stage_work(k, m, n, d, args.method, level)), key=lambda k: stages[k])
    flops, bytes_, bound = stage_work(dom, m, n, d, args.method, level)
    if dom in ("trsm", "trsm_gram") and trsm_blocked:
        # the dominant kernel is the DMMA leaf solve (2 launches per solve at n = 2048):
        # one leaf launch of the solve's shape, timed live with CUDA events (on a 1M-row
        # slice when A_p is chunked: there is no room for a full-height output)
        leaves, _ = trsm_blocks(n)
        lm = m if dom == "trsm" else min(m, 1 << 20)
        leaf_ms = time_trsm_leaf(a[:lm], lm, n, leaves[0]) * (m / lm)
        peak, src = fp64_peak()
        lf = float(m) * leaves[0] ** 2
        achieved = lf / (leaf_ms * 1e-3) / 1e12
        roof = {"kernel": "trsm leaf (trsm_kernel, m x %d of the blocked TRSM)" % leaves[0], "bound": "tensor",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": ncu_traffic("trsm_leaf"), "peak_source": src, "algorithmic_flops": lf,
                "launch_ms": leaf_ms, "launches_per_solve": len(leaves),
                "stage_frac": trsm_roofline(m, n, True) * 1e3 / stages[dom] if dom == "trsm" else None,
                "pipe": "FP64 DMMA (mma.sync m8n8k4); updates on INT8 tcgen05 (Ozaki-II)"}
    elif bound == "tensor" and ozaki and dom in ("gram", "kappa0"):
        peak, src = int8_peak()
        ops = gram_moduli(m) * flops   # exact INT8 products (15 moduli at 4M rows) of the FP64 SYRK / GEMM
        achieved = ops / (stages[dom] * 1e-3) / 1e12
        roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s",
                "frac": achieved / peak, "traffic": ncu_traffic(dom), "peak_source": src,
                "algorithmic_ops": ops, "pipe": "INT8 tcgen05 kind::i8 (16-modulus Ozaki-II FP64 emulation)"}
    elif bound == "tensor":
        peak, src = fp64_peak()
        achieved = flops / (stages[dom] * 1e-3) / 1e12
        roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": ncu_traffic(dom), "peak_source": src,
                "algorithmic_flops": flops, "pipe": "FP64 DMMA (mma.sync m8n8k4)"}
    else:
        peak, src = hbm_peak()
        achieved = bytes_ / (stages[dom] * 1e-3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(dom), "peak_source": src,
                "algorithmic_bytes": bytes_}
    per_stage = {}
    for k, v in stages.items():
        w = stage_work(k, m, n, d, args.method, level)
        if w and w[2] == "tensor":
            per_stage[k] = {"ms": v, "tflops": w[0] / (v * 1e-3) / 1e12}
        elif w:
            per_stage[k] = {"ms": v, "gbs": w[1] / (v * 1e-3) / 1e9}
        else:
            per_stage[k] = {"ms": v}
    fp64_total = (m * n * n if args.precision == "auto" else 0) + m * n * n + \
        (2.0 if args.method == "hpne" else 1.0) * m * n * n
    t_roof_fp64 = fp64_total / (fp64_peak()[0] * 1e12) + 2 * 8.0 * m * n / (hbm_peak()[0] * 1e9)
    eng = engine_roofline(m, n, d, args.method, args.precision == "auto", ozaki, trsm_blocked)
    t_roof = sum(eng.values())

    # ---- e2e: host buffers, H2D + D2H inside the timed region ----
    e2e = None
    host_need = 8.0 * m * n * world * 1.15
    host_ok = True
    try:
        import psutil
        host_ok = psutil.virtual_memory().available > host_need
    except Exception:  # noqa: BLE001
        pass
    if not host_ok:
        e2e = {"value": None, "unit": "ms", "skipped": f"host RAM: {world} pinned shards need {host_need / 1e9:.0f} GB"}
    elif not args.no_e2e and args.e2e_steps > 0:
        a_host = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
        a_host.copy_(a)
        b_host = b.to("cpu").pin_memory()
        del a, rep, reps
        torch.cuda.empty_cache()
        solve(a_host, b_host)          # untimed: first device allocations of the H2D target
        torch.cuda.synchronize()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.e2e_steps):
            r2 = solve(a_host, b_host)
        f1.record()
        torch.cuda.synchronize()
        barrier()
        e2e_ms = f0.elapsed_time(f1) / args.e2e_steps
        if dist is not None:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 8 * m * n + 8 * m,
               "d2h_bytes_per_step": 8 * n + 16, "steps": args.e2e_steps,
               "rel_error": r2.relative_error, "host_buffers": "pinned torch CPU tensors"}
        if not args.no_e2e_pageable and world == 1:
            # the reference's own convention: pageable numpy arrays in, numpy x_hat out
            import numpy as np
            a_np = np.empty((m, n), dtype=np.float64)
            np.copyto(a_np, a_host.numpy())
            b_np = b_host.numpy().copy()
            del a_host
            torch.cuda.synchronize()
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            g0.record()
            r3 = solve(a_np, b_np)
            g1.record()
            torch.cuda.synchronize()
            e2e["pageable_numpy"] = {"value": g0.elapsed_time(g1), "unit": "ms", "steps": 1,
                                     "rel_error": r3.relative_error,
                                     "note": "A and b as pageable numpy arrays (src/solvers.py convention)"}
            del a_np, b_np

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            ref = CpuReference(args)
            v = ref.step()
            cpu = {"value": v, "unit": "ms", "cores": cpu_cores(), "kind": "port", "sample": ref.describe(),
                   "measured_seconds": ref.spent, "stages_s": ref.last["full_s"]}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "ms", "cores": cpu_cores(), "kind": "port", "sample": f"failed: {ex!r}"}
    extra = {}
    if world == 1 and not args.no_config1:
        try:
            extra["config1_latency"] = config1_latency()
        except Exception as ex:  # noqa: BLE001 -- an extra report; never fails the bench line
            extra["config1_latency"] = {"error": repr(ex)}
    if world == 1 and m == CONFIG3_M:
        extra["config4_t1_extrapolated_ms"] = {
            "value": 4 * ms, "basis": "linear-in-m extrapolation 4 x T(1 GPU, 4M x 2048): config 4 "
                                      "(16M x 2048, 275 GB) does not fit one GPU (SURVEY §8(d))"}
    line = {"metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong" if world > 1 else "weak", **extra,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (GPU Algorithm-2 generator, probgen.py)",
            "config": workload_config(args), **summary,
            "roofline": roof,
            "roofline_solve": {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms,
                               "stages_roof_ms": {k: v * 1e3 for k, v in eng.items()},
                               "model": (("blocked TRSM: DMMA leaves m nl^2 / FP64 DMMA peak + INT8 updates "
                                          "(16 products / INT8 peak + residue and reconstruction passes / HBM)"
                                          if trsm_blocked else "TRSM m n^2 / FP64 DMMA peak") +
                                         "; kappa0 SYRK + Gram as 16 INT8 "
                                         "products / measured INT8 peak + residue/column passes / HBM"
                                         if ozaki else "FP64 flops / measured DGEMM peak") +
                                        "; sketch 2dmn / fp16 peak; residual 8mn / HBM",
                               "t_roof_fp64_only_ms": t_roof_fp64 * 1e3,
                               "frac_vs_fp64_only": t_roof_fp64 * 1e3 / ms},
            "stages_ms": per_stage, "other_method": other_line, "e2e": e2e, "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / args.steps, "clocks": clk}
    print(json.dumps(line), flush=True)


def config1_latency(reps=50):
    """Config 1 (1000 x 100, kappa 1e8, rho 1e-6; the reference's CPU-runnable case, HPNE
    "single") per-solve latency from device arrays: the eager algorithm1_pipeline against
    one PipelinePlan graph replay (deferred verdicts).  Host wall time per solve including
    the result read (the solve is latency-bound); an extra report, not the headline."""
    import torch
    import paper_2603_16644_b200 as sq
    from paper_2603_16644_b200.probgen import generate_problem_device
    a, b, _ = generate_problem_device(1000, 100, 1e8, 1e-6, 11)
    out = {"config": "1000 x 100, kappa 1e8, rho 1e-6, hpne, precision single, device arrays", "reps": reps}
    plan = sq.PipelinePlan(1000, 100, method="hpne", precision="single", seed=1)

    def eager():
        return sq.algorithm1_pipeline(a, b, "hpne", "single", seed=1, diagnostics=False)

    for name, fn in (("eager_ms", eager), ("graph_ms", lambda: plan.solve(a, b))):
        for _ in range(5):
            rep = fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            rep = fn()
        torch.cuda.synchronize()
        out[name] = (time.perf_counter() - t) / reps * 1e3
        out[name.replace("_ms", "_x")] = rep.x_hat
    out["x_bitwise_equal"] = bool((out.pop("eager_x") == out.pop("graph_x")).all())
    return out


def rep_kappa0(rep):
    d = rep.precision_decision
    if d is None or (isinstance(d.kappa0, float) and math.isnan(d.kappa0)):
        return None
    return d.kappa0


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":      # the CPU arm runs on rank 0 only anyway
            run_reference(args, 0, 1)
            return 0
        # plain `python bench.py --gpus N`: spawn one rank per GPU ourselves
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"metric": METRIC, "n_gpus": args.gpus,
                              "error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}"}))
            return 1
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return 0
    run_ours(args, rank, world)
    return 0


if __name__ == "__main__":
    sys.exit(main())
