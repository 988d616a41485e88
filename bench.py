#!/usr/bin/env python
"""LSRN hot-path benchmark (driver contract).

One step = one full LSRN solve of the configured workload on device-resident
inputs: Gaussian sketch (K1 G tiles + K2 DMMA) -> [NCCL allreduce] -> SVD (cuSOLVER,
outside the hot path, reported separately) -> N -> fused LSQR (or CS)
iterations (K5/K6/K8, one CUDA graph) -> x.

Default workload: BASELINE.json's largest single-GPU configuration, c5: dense
1e6 x 1e4 (80 GB, column scales 1 -> 1e-5), gamma = 2 (s = 2e4), LSQR with the
predictable Thm 4.5 count (96 iterations), row-sharded over N GPUs.  A is far
larger than L2 (126 MB), so no L2 flush is needed between steps.  The other
configs (--config c1..c4, t4) are parity-test cases and optional bench lines.

  python bench.py [--gpus N --steps K --warmup W] [--config c5] [--solver lsqr|cs]
  python bench.py --impl reference ...     # the CPU oracle arm (rank 0 only)
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "lsrn_solve_s"
UNIT = "s"
FP64_PEAK_TFLOPS = 37.2     # DMMA.8x8x4 sustained 12 s at 1965 MHz (profiles/r02_fp64_sustained.jsonl)
FP64_PEAK_NOTE = ("fp64 DMMA peak measured on this pool's B200 (MEASURED_PEAKS.json has no fp64 entry): "
                  "mma.sync m8n8k4 back to back for 12 s, 37.2 TFLOP/s at 1965 MHz, no throttle "
                  "(tools/microbench/fp64_sustained.cu, profiles/r02_fp64_sustained.jsonl; burst 36.9, "
                  "cuBLAS DGEMM 8192^3 sustained 35.5)")
DFMA_PEAK_TFLOPS = 36.8     # DFMA (FP64 ALU) peak measured by the same microbenchmark
DFMA_PEAK_NOTE = "fp64 DFMA peak measured by tools/microbench/fp64_peak.cu (profiles/r01_fp64_peak.jsonl)"


def load_traffic(workload):
    """DRAM bytes per launch of the dominant kernels from one committed ncu --set full
    capture (profiles/traffic.json, written by tools/ncu_summary.py traffic); None if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload, {})
    except Exception:
        return {}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.first = 0

    def mark(self):
        """Start of the timed region: samples before it (sampler start-up) are dropped."""
        self.first = len(self.lines)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines[self.first:] or self.lines
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def host_info():
    """CPU model, cores and RAM of the host the oracle runs on (BASELINE.md's plan asks for them)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemTotal"):
                    ram = round(int(ln.split()[1]) / 1024 ** 2, 1)
                    break
    except OSError:
        pass
    return {"cpu": model, "nproc": os.cpu_count(), "ram_gb": ram}


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


def cpu_baseline(cfg_name, solver, sample_rows=1024, svd_k=2000, full_max=2.5e8):
    """The oracle (as it stands, oracle/) timed on the box's host cores.

    Small configs (k <= 2048 and L k <= 2.5e8: c1, c2) are solved IN FULL by the oracle
    and the wall time is the value.  Larger ones are timed stage by stage on bounded
    pieces of the same workload and scaled by the stage's operation count:
      sketch  oracle.sketch.sketch on the first `sample_rows` long-index rows of the
              config's own matrix (same recipe bytes), x L / rows      (2 s k L flops);
      SVD     oracle.precond.factor on a Gaussian s' x k' sketch with k' = svd_k,
              s' = ceil(gamma k'), x (k / k')^3                       (2 s k^2 + 11 k^3, s = gamma k);
      iters   three passes of the oracle's operator pair (A N y, N^T A^T u) with the
              row sample and a full k x k N, per pass = t_A L / rows + t_N, x passes.
    """
    import math
    import numpy as np
    from oracle import bounds
    from oracle.lsrn import LongOperator
    from oracle.lsrn import solve as orc_solve
    from oracle.precond import factor
    from oracle.sketch import plan as orc_plan
    from oracle.sketch import sketch as orc_sketch
    from synth.generate import CONFIGS, SKETCH_SEED, make_problem
    cfg = CONFIGS[cfg_name]
    m, n = cfg["m"], cfg["n"]
    L, k = max(m, n), min(m, n)
    t0 = time.perf_counter()
    if k <= 2048 and L * k <= full_max:
        p = make_problem(cfg_name)
        A = p.to_scipy() if p.kind == "csr" else p.dense_A().numpy()
        rep = orc_solve(A, p.b.numpy(), gamma=cfg["gamma"], lam=cfg["lam"], solver=solver)
        wall = time.perf_counter() - t0
        return {"value": rep["t_sketch"] + rep["t_svd"] + rep["t_iter"], "unit": UNIT, "cores": _blas_threads(),
                "kind": "oracle", "host": host_info(),
                "sample": (f"the full {cfg_name} solve ({solver}) by the oracle: sketch {rep['t_sketch']:.1f}s "
                           f"svd {rep['t_svd']:.1f}s iterations {rep['t_iter']:.1f}s ({rep['iters']} it.)"),
                "stages_s": {"sketch": rep["t_sketch"], "svd": rep["t_svd"], "iterations": rep["t_iter"]},
                "sample_wall_s": wall}
    pl = orc_plan(m, n, cfg["gamma"], cfg["lam"])
    s = pl["s"]
    rows = min(sample_rows, L)
    p = make_problem(cfg_name, shard=(0, rows))
    import scipy.sparse as sp
    if p.kind == "csr":
        X = sp.csr_matrix((p.val.numpy(), p.colind.numpy(), p.rowptr.numpy()), shape=(rows, k))
    else:
        X = p.X.numpy()
    ta = time.perf_counter()
    orc_sketch(X, s, SKETCH_SEED, pl["sigma_x"], 0.0)
    t_sk = (time.perf_counter() - ta) * L / rows
    # SVD: the oracle's factor() of the sketch of a k' = svd_k column instance of the same
    # recipe (same column / row scaling, so the same conditioning: the Jacobi sweep count
    # depends on it), then scaled by (k / k')^3 at fixed gamma
    kp = min(svd_k, k)
    sp_ = int(math.ceil(cfg["gamma"] * kp))
    ps = make_problem(cfg_name, m=2 * sp_, n=kp) if m >= n else make_problem(cfg_name, m=kp, n=2 * sp_)
    Xs = (sp.csr_matrix((ps.val.numpy(), ps.colind.numpy(), ps.rowptr.numpy()), shape=(2 * sp_, kp))
          if ps.kind == "csr" else ps.X.numpy())
    Ats = orc_sketch(Xs, sp_, SKETCH_SEED, 1.0, 0.0)
    ta = time.perf_counter()
    factor(Ats)
    t_svd = (time.perf_counter() - ta) * (k / kp) ** 3
    del Xs, Ats, ps
    r = k
    alpha = bounds.default_alpha(s)
    sl, su = bounds.sigma_bounds(s, r, alpha)
    passes = bounds.lsqr_count(1e-14, r, s) + 1 if solver == "lsqr" else bounds.cs_passes(sl, su, 1e-14)
    op = LongOperator(X, pl["sigma_x"], 0.0)
    Nm = np.random.default_rng(1).standard_normal((k, k))
    y, u = np.ones(k), np.ones(rows)
    ta = time.perf_counter()
    for _ in range(3):
        op.PT(op.P(y) + u)
    t_a = (time.perf_counter() - ta) / 3
    ta = time.perf_counter()
    for _ in range(3):
        Nm.T @ (Nm @ y)
    t_n = (time.perf_counter() - ta) / 3
    del Nm
    t_it = passes * (t_a * L / rows + t_n)
    wall = time.perf_counter() - t0
    return {"value": t_sk + t_svd + t_it, "unit": UNIT, "cores": _blas_threads(), "kind": "oracle",
            "host": host_info(),
            "sample": (f"oracle stages on pieces of {cfg_name} scaled by operation count: sketch of the first "
                       f"{rows} of L={L} rows x{L / rows:.0f} ({t_sk:.0f}s); SVD (factor) of the {sp_}x{kp} sketch of a "
                       f"{kp}-column instance of the recipe "
                       f"x(k/{kp})^3 ({t_svd:.0f}s); {passes} passes of the operator pair, long side x{L / rows:.0f} "
                       f"plus a {k}x{k} N ({t_it:.0f}s)"),
            "stages_s": {"sketch": t_sk, "svd": t_svd, "iterations": t_it},
            "sample_wall_s": wall}


def run_reference(args):
    """--impl reference: the CPU oracle arm (rank 0 only, N > 1 ranks exit 0).  Each step is
    one bounded oracle measurement of the workload (cpu_baseline); value = the median."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    last = None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        last = cpu_baseline(args.config, args.solver, sample_rows=args.ref_rows, svd_k=args.ref_svd_k)
        vals.append(last["value"])
    wall = time.perf_counter() - t0
    v = statistics.median(vals)
    cb = dict(last)
    cb["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "solver": args.solver},
            "note": ("value = the oracle's time for the whole workload, estimated per step from a bounded "
                     f"sample (cpu_baseline.sample); the {args.steps} samples took {wall:.0f} s of wall time"),
            "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "t4"])
    ap.add_argument("--solver", default="lsqr", choices=["lsqr", "cs"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=512)
    ap.add_argument("--ref-svd-k", type=int, default=1024)
    ap.add_argument("--cpu-rows", type=int, default=1024)
    ap.add_argument("--cpu-svd-k", type=int, default=2000)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1109_5981_b200 import dist as lsrn_dist
    from paper_1109_5981_b200 import lsrn
    from synth.generate import CONFIGS, SKETCH_SEED, make_problem

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    m, n = cfg["m"], cfg["n"]
    L = max(m, n)
    lo, hi = lsrn_dist.shard_bounds(L, world, rank)
    p = make_problem(args.config, device=dev, shard=(lo, hi) if world > 1 else None)
    csr = p.kind == "csr"
    X = lsrn.Csr(p.rowptr, p.colind, p.val) if csr else p.X
    b = p.b
    stream = torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    ctx = lsrn_dist.context(stream=stream)
    ctx.set_profiling(True)
    kw = dict(solver=args.solver, gamma=cfg["gamma"], lam=cfg["lam"], tol=1e-14, seed=SKETCH_SEED, lo=lo,
              cnt=hi - lo)
    with torch.cuda.stream(stream):
        x, rep = ctx.solve(X, b, m, n, **kw)
        for _ in range(max(0, args.warmup - 1)):
            x, rep = ctx.solve(X, b, m, n, **kw)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the sampler starts before the timed region (nvidia-smi's start-up would
    # otherwise stall the first timed solves) and keeps sampling through it
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(1.0)
    barrier()
    clocks.mark()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps, stats = [], []
    torch.cuda.nvtx.range_push("lsrn_step")
    torch.cuda.profiler.start()      # ncu --profile-from-start off captures only the timed steps
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            x, rep = ctx.solve(X, b, m, n, **kw)
            reps.append(rep)
        e1.record(stream)
    torch.cuda.profiler.stop()
    torch.cuda.nvtx.range_pop()
    barrier()
    # per-kernel event times of the last timed step (read after the timed region: the
    # library keeps the events, so no host work sits between the timed solves)
    stats.append(ctx.stats())
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    # ---- per-stage and per-kernel numbers (medians over the timed steps)
    def med(key, src):
        return statistics.median(float(r[key]) for r in src)

    t_sketch = med("t_sketch", reps)
    t_svd = med("t_svd", reps)
    t_iter = med("t_iter", reps)
    t_ar = med("t_allreduce", reps)
    sk_ms = med("sketch_ms", stats)
    lp_ms = med("long_pass_ms", stats)
    launches = int(statistics.median(s["launches"] for s in stats))
    s_ = reps[-1]["s"]
    k = min(m, n)
    cnt = hi - lo
    nnz = int(p.val.numel()) if csr else cnt * k
    sketch_flops = 2.0 * s_ * nnz
    peaks, peak_src = load_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # algorithmic bytes of one long pass, from the library: dense 8k+16 per row;
    # CSR 12 per nonzero + 24 per row + 12 per light-CSC entry
    lp_bytes = statistics.median(float(st["long_pass_bytes"]) for st in stats)
    sketch_tf = sketch_flops / (sk_ms * 1e-3) / 1e12
    lp_gbs = lp_bytes / (lp_ms * 1e-3) / 1e9 if lp_ms > 0 else None
    iters = reps[-1]["iters"]
    # dominant kernel by share of the step
    sketch_share = (sk_ms / 1e3) / (ms / 1e3)
    lp_share = (lp_ms / 1e3) * max(iters + 1, 1) / (ms / 1e3)
    if csr:
        roof_sketch = {"kernel": "csr_gen_g_kernel + csr_sketch_heavy_mma_kernel + csr_sketch_light_g_kernel (K4 "
                                 "stored G per chunk; the light gathers are bound by L2-to-SM traffic, 8 B of G "
                                 "per (nonzero, sketch row), not by FP64 issue: DESIGN.md §6 K4 round 2c)",
                       "bound": "alu",
                       "achieved": sketch_tf, "peak": DFMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                       "frac": sketch_tf / DFMA_PEAK_TFLOPS, "traffic": None,
                       "algorithmic": f"2*s*nnz = {sketch_flops:.4g} flop per sketch (+ s*cnt normals, not counted)",
                       "peak_source": DFMA_PEAK_NOTE, "share_of_step": sketch_share}
    else:
        roof_sketch = {"kernel": "sketch_gen_g_kernel + sketch_ws_kernel (K1 once per launch into stored G "
                                 "tiles, K2 DMMA warp-specialized; the sketch stage)", "bound": "tensor",
                       "achieved": sketch_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                       "frac": sketch_tf / FP64_PEAK_TFLOPS, "traffic": None,
                       "algorithmic": f"2*s*k*L = {sketch_flops:.4g} flop per sketch stage (all its launches)",
                       "peak_source": FP64_PEAK_NOTE, "share_of_step": sketch_share}
    roof_lp = {"kernel": "csr_rowdot + csr_colgather (K6-CSR)" if csr else "rowpass_bulk_kernel long pass (K6)",
               "bound": "hbm", "achieved": lp_gbs, "peak": hbm_peak,
               "unit": "GB/s", "frac": (lp_gbs / hbm_peak) if lp_gbs else None, "traffic": None,
               "algorithmic": f"{lp_bytes:.4g} B per pass ({'12 nnz + 24 rows (+ 12 light-CSC if k > 2048)' if csr else 'rows*(8k+16)'})",
               "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})", "share_of_step": lp_share}
    traffic = load_traffic(args.config)
    roof_sketch["traffic"] = traffic.get("sketch")
    roof_lp["traffic"] = traffic.get("long_pass")
    if traffic:
        roof_sketch["traffic_source"] = roof_lp["traffic_source"] = traffic.get("source")
    roofline = roof_sketch if sketch_share >= lp_share else roof_lp

    # ---- end to end through the C ABI with HOST buffers (H2D of A, b and D2H of x inside)
    e2e = None
    if not args.no_e2e:
        def pinned(t):          # straight into pinned host memory (c5's A is 80 GB: no pageable copy)
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h
        if csr:
            Xh = lsrn.Csr(pinned(p.rowptr), pinned(p.colind), pinned(p.val))
            h2d_A = int(p.rowptr.numel() * 8 + p.colind.numel() * 4 + p.val.numel() * 8)
        else:
            Xh = pinned(X)
            h2d_A = int(Xh.numel() * 8)
        bh = pinned(b)
        # the device copy of A is not used by the end-to-end solves (they stage A from the
        # host into the workspace): free it so the staging copy fits next to it
        X = p.X = p.val = p.colind = p.rowptr = None
        ctx._ws = None
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        nsteps = min(args.e2e_steps, args.steps)
        barrier()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ctx.solve(Xh, bh, m, n, host_io=True, **kw)
            barrier()
            h0.record(stream)
            for _ in range(nsteps):
                xh, _r = ctx.solve(Xh, bh, m, n, host_io=True, **kw)
            h1.record(stream)
        barrier()
        ems = h0.elapsed_time(h1) / nsteps
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": float(te.item()) / 1e3, "unit": UNIT,
               "h2d_bytes_per_step": h2d_A + int(bh.numel() * 8),
               "d2h_bytes_per_step": int(xh.numel() * 8),
               "steps": nsteps}
        del Xh, bh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.config, args.solver, sample_rows=args.cpu_rows, svd_k=args.cpu_svd_k)
        except Exception as ex:  # report, do not fail the bench
            cpu = {"error": repr(ex)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms / 1e3, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "shape": [m, n], "s": s_, "r": reps[-1]["r"],
                       "solver": args.solver, "iters": iters, "gamma": cfg["gamma"], "lambda": cfg["lam"],
                       "tol": 1e-14, "parallelism": f"row-shard x{world}" if m >= n else f"col-shard x{world}",
                       "l2": "inputs larger than L2 (A = %.2f GB), no flush" % (
                           (nnz * 12 + cnt * 8) / 1e9 if csr else cnt * k * 8 / 1e9)},
            "stages_s": {"sketch": t_sketch, "allreduce": t_ar, "svd": t_svd, "iterations": t_iter,
                         "hot_path_excl_svd": t_sketch + t_ar + t_iter},
            "sketch_tflops": sketch_tf, "matvec_gbs": lp_gbs,
            "roofline": roofline, "roofline_kernels": {"sketch": roof_sketch, "long_pass": roof_lp},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches * args.steps,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
