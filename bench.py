#!/usr/bin/env python
"""Benchmark of the fused fp64 SGN split-form BS3 stage pipeline on B200.

Metric (BASELINE.json): grid-point RK-stage updates per second on an 8192^2
fp64 grid (config 4: periodic [-1,1]^2, manufactured bathymetry and state at
t = 0.3, lambda = 500, fixed dt = 0.25 dx / 20), plus achieved HBM GB/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--bc periodic|reflecting] [--scaling weak|strong] [--config5]
                    [--n NX] [--rows R] [--sustained S]

* ``value``   : point-stage updates/s, device time (CUDA events on the
                library stream, max over ranks) of one hsgn_bs3_fixed_steps
                call of K graph-captured fused steps, in place on resident
                states; every state is >= 2.7 GB (> 126 MB L2), so no L2
                flush is needed between steps.
* ``e2e``     : the same metric through the public API with HOST buffers:
                upload of the pinned host state, one ``adaptive_solve`` call
                (fixed dt, K steps, incl. its initial RHS) and the download of
                the result, all inside the wall-clock window (device buffers
                allocated before it).
* ``roofline``: the dominant kernel S12 (stages 1 + 2)
                on SURVEY section 8(d)'s roofline: 128 B per point-stage x the
                2 point-stages S12 updates per node, over its mean launch time
                measured by CUDA event nodes inside the timed graphs; with its
                own-byte HBM fraction and its FP64-pipe fraction beside it.
* ``sustained``: the same measurement over S steps (default 300, ~1.3 s):
                the power-capped long-run rate.
* ``cpu_baseline``: the reference CPU path (oracle/_ref, the unmodified
                reference compiled in place; else the C oracle port) on this
                host's cores, on the same workload (all threads, median of
                reps) plus a 1-thread line on a 2048^2 slice.
Multi-GPU: ``--gpus N`` outside torchrun launches N ranks itself
(torch.distributed.run; it refuses when fewer than N GPUs are visible); each
rank owns a y-slab, halos and the step agreement go over NCCL inside the
captured graphs.  Weak scaling (default): every rank owns an NX x R slab of
an NX x (R N) grid (default 8192 x 8192, the config-4 block; --config5:
16384 x 4096); strong: a fixed NX x NY grid (default 16384^2 at N > 1).
``--impl reference`` runs the reference CPU implementation only on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_POINT_STAGE = 128  # unfused compulsory traffic per grid-point RK stage
OWN_BYTES_PER_NODE = {"S12": 128, "S3": 88}  # y, k1, b -> ynew; ynew, b -> k4
POINT_STAGES_PER_NODE = {"S12": 2, "S3": 1}
# FP64 instructions (DADD + DMUL + DFMA) per node of each kernel, from the ncu
# SASS mixes in profiles/ (the compute roofline of the FP64-issue-bound kernels)
FP64_PER_NODE = {"S12": 420.4, "S3": 180.7}
FP64_SOURCE = "profiles/r2f_sass_mix_s12.txt, profiles/r2f_sass_mix_s3.txt"
FP64_LANES_PER_SM, N_SM = 64, 148
METRIC = "grid-point RK-stage updates/sec on 8192² fp64 grid; achieved HBM GB/s"
UNIT = "point-stage updates/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture (profiles/traffic.json), with its source."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as fh:
        d = json.load(fh)
    return d.get(kernel), d.get("_source")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region:
    sampling starts before and stops after it, and only the samples stamped
    inside [start(), stop()] (the timed call) enter the summary."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")
    # cumulative microseconds each limiter held the clocks down: the delta
    # over the timed call catches a limiter between two instantaneous samples
    CQ = ("clocks_event_reasons_counters.sw_power_cap,clocks_event_reasons_counters.sw_thermal_slowdown,"
          "clocks_event_reasons_counters.hw_thermal_slowdown,clocks_event_reasons_counters.hw_power_brake_slowdown")
    CNAMES = ("sw_power_cap", "sw_thermal_slowdown", "hw_thermal_slowdown", "hw_slowdown")

    def __init__(self, index=0, period_ms=20):
        self.index = index
        self.period_ms = period_ms
        self.samples = []
        self._p = None
        self._t0 = self._t1 = None
        self._c0 = self._c1 = None

    def _counters(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.CQ}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
            return [float(v) for v in out.strip().split(",")]
        except Exception:
            return None

    def start(self):
        import datetime
        self._c0 = self._counters()
        self._t0 = datetime.datetime.now()

    def stop(self):
        import datetime
        self._t1 = datetime.datetime.now()
        self._c1 = self._counters()

    def __enter__(self):
        try:  # one long-running nvidia-smi sampling every period_ms (started before, killed after)
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", f"-lms={self.period_ms}"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the first sample land before the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.1)
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=10)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        import datetime
        rows = []
        for line in out.strip().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 8:
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                except ValueError:
                    ts = None
                rows.append((ts, parts[1:]))
        inside = [p for ts, p in rows if ts and self._t0 and self._t1 and self._t0 <= ts <= self._t1]
        self.samples = inside if len(inside) >= 2 else [p for _, p in rows]
        self.windowed = len(inside) >= 2

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        sm = [x for x in (num(s[0]) for s in self.samples) if x is not None]
        mx = [x for x in (num(s[1]) for s in self.samples) if x is not None]
        pw = [x for x in (num(s[6]) for s in self.samples) if x is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = {names[k] for s in self.samples for k in range(4) if "Active" in s[2 + k] and "Not" not in s[2 + k]}
        held = {}
        c0, c1 = self._c0, self._c1
        if c0 and c1 and len(c0) == len(c1) == 4:
            for k, nm in enumerate(self.CNAMES):
                if c1[k] > c0[k]:
                    reasons.add(nm)
                    held[nm + "_ms"] = (c1[k] - c0[k]) / 1e3
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "limiter_ms": held, "power_w_median": statistics.median(pw) if pw else None,
                "samples": len(self.samples),
                "window": "timed call only" if getattr(self, "windowed", False) else "whole sampler run"}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def keep_heap():
    """glibc: serve the reference's field allocations from the heap and never
    trim it, so a solve reuses the pages the previous one touched instead of
    page-faulting its ~44 GB workspace (8192^2) anew.  The reference
    allocates its workspace per adaptive_solve call; in its own CLI that is
    once per run, amortised over thousands of steps -- this keeps a short
    timed solve representative of that.  (Allocator tuning of this process
    only; the reference code is unchanged.)"""
    import ctypes
    try:
        libc = ctypes.CDLL("libc.so.6")
        libc.mallopt(-4, 0)   # M_MMAP_MAX: no mmap'ed chunks
        libc.mallopt(-1, -1)  # M_TRIM_THRESHOLD: never trim the heap top
    except Exception:
        pass


class CpuReference:
    """The reference CPU implementation of the path on this host's cores:
    oracle/_ref (the unmodified reference headers compiled in place; OpenMP)
    when it was built, else the C oracle port.  A "step" is one fixed-step
    BS3 step (time_integration.hpp:262-345: 3 RHS + stage axpys + min-h) of
    the same workload (same closed-form input)."""

    def __init__(self, bc: str, nx: int, ny: int, threads: int = 0):
        keep_heap()
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_lib import Oracle, Phys, default_cfg, make_grid as omake, ref_available
        from paper_2601_02540_b200.workloads import bench_case
        self.kind = "reference" if ref_available() else "port"
        self.orc = Oracle("ref" if self.kind == "reference" else "orc")
        self.cores = threads or (os.cpu_count() or 1)
        self.orc.set_threads(self.cores)
        self.nx, self.ny, self.bc = nx, ny, bc
        g, self.q, self.b, lam, self.dt, aux = bench_case(bc, nx, ny)
        kx = ky = 1 if bc == "reflecting" else 0
        self.og = omake(nx, ny, g.x_min, g.x_max, g.y_min, g.y_max, kx, ky)
        if aux:  # w, eta = init_auxiliary (model.hpp:93-105), the reference's own
            self.q = self.orc.init_auxiliary(self.og, self.b, self.q)
        self.ph = Phys(9.81, lam, 1e-12)
        self.cfg = default_cfg

    def steps(self, k: int) -> float:
        """Wall seconds of k fixed steps, minus the initial tendency the
        solve evaluates first (its share of the 3k + 1 evaluations)."""
        t0 = time.perf_counter()
        _, rec = self.orc.solve(self.og, self.ph, self.b, self.q, 0.0, k * self.dt, self.cfg(fixed_dt=self.dt))
        el = time.perf_counter() - t0
        assert rec.accepted == k and not rec.aborted
        return el * (3 * k) / (3 * k + 1)

    def rate(self, k, seconds):
        return 3 * k * self.nx * self.ny / seconds


def cpu_baseline(bc: str, nx: int, ny: int, reps: int = 3, steps: int = 2):
    """cmd_bench-style (cli.hpp:248-268) median of reps on the full workload
    with every host thread, plus a 1-thread line on a 2048^2 slice."""
    ref = CpuReference(bc, nx, ny)
    ref.steps(1)  # warm-up: page-in, OpenMP pool, first touch of the workspace
    secs = [ref.steps(steps) for _ in range(reps)]
    med = statistics.median(secs)
    n1 = min(2048, nx)
    one = CpuReference(bc, n1, n1, threads=1)
    t1 = one.steps(1)
    return {"value": ref.rate(steps, med), "unit": UNIT, "cores": ref.cores, "kind": ref.kind, "cpu": cpu_model(),
            "sample": f"the full {nx}x{ny} {bc} workload, {steps} fixed BS3 steps per rep via the reference "
                      f"adaptive_solve(fixed_dt), median of {reps} reps ({', '.join(f'{s:.2f}' for s in secs)} s) "
                      f"on {ref.cores} OpenMP threads",
            "one_thread": {"value": one.rate(1, t1), "cores": 1,
                           "sample": f"{one.nx}x{one.ny} slice, 1 fixed step, {t1:.2f} s"}}


def shapes(args, world: int):
    """(nx, global ny, scaling) of the run."""
    if args.scaling == "strong":
        nx = args.n or (16384 if args.config5 or world > 1 else 8192)
        return nx, args.ny or nx, "strong"
    nx = args.n or (16384 if args.config5 else 8192)
    rows = args.rows or (4096 if args.config5 else nx)
    return nx, rows * world, "weak"


def workload_config(args, nx: int, ny: int, world: int, scaling: str) -> dict:
    bc = args.bc
    if world > 1 or args.config5:
        what = f"config 5 ({scaling} scaling)"
    elif bc == "periodic":
        what = "config 4" if nx == ny == 8192 else "config-4 input"
    else:
        what = "config-3/5 reflecting walls"
    if bc == "periodic":
        desc = (f"{what}: {nx}x{ny} periodic, manufactured bathymetry + state (t=0.3) on "
                f"[-1,1]x[-1,{-1 + 2 * ny / nx:g}], lambda=500, fixed-step BS3 dt=0.25dx/20")
    else:
        desc = (f"{what}: {nx}x{ny} reflecting walls, gaussian_obstacle(bounded) on [-5,35]x[-10,10], lambda=500, "
                f"fixed-step BS3 dt=0.25min(dx,dy)/20")
    return {"workload": desc, "bc": bc, "grid": f"{nx}x{ny}", "points": nx * ny, "scaling": scaling,
            "parallelism": f"slab{world}" if world > 1 else "1 GPU, whole grid"}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation, timed per
    step on this host's cores (rank 0 only under torchrun), on the same
    workload as the device arm (the full grid up to the 8192^2 config-4 size,
    which needs ~44 GB of reference workspace; beyond it one rank's share)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = max(1, args.gpus)
    nx, ny, scaling = shapes(args, world)
    ny_ref = ny if nx * ny <= 8192 * 8192 else max(4, ny // world)
    ref = CpuReference(args.bc, nx, ny_ref)
    ref.steps(max(1, args.warmup))  # warm-up steps (page-in, OpenMP pool, workspace first touch)
    total = ref.steps(args.steps)   # K steps in one solve, as the reference integrates
    v = ref.rate(args.steps, total)
    cb = {"value": v, "unit": UNIT, "cores": ref.cores, "kind": ref.kind, "cpu": cpu_model(),
          "sample": f"{nx}x{ny_ref} of the {args.bc} workload, {args.steps} fixed BS3 steps in one reference "
                    f"adaptive_solve(fixed_dt) ({total:.2f} s) after {max(1, args.warmup)} warm-up steps, "
                    f"{ref.cores} OpenMP threads"}
    cfg = workload_config(args, nx, ny, world, scaling)
    cfg.update(parallelism="cpu-openmp", reference_grid=f"{nx}x{ny_ref}", same_config=(ny_ref == ny))
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference", "config": cfg, "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def visible_gpus() -> int:
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30).stdout
        return sum(1 for line in out.splitlines() if line.startswith("GPU "))
    except Exception:
        return 0


def refuse(args, n_dev: int) -> int:
    """Fewer GPUs than --gpus asks for: say so and exit 2 (never time fewer
    GPUs than the line reports)."""
    sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, this node has {n_dev}; "
                     f"refusing to time fewer GPUs than requested\n")
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"metric": METRIC, "n_gpus": args.gpus,
                          "error": f"--gpus {args.gpus} requested, {n_dev} GPU(s) visible"}), flush=True)
    return 2


def self_launch(args) -> int:
    """--gpus N > 1 outside torchrun: start N ranks (one per GPU) with
    torch.distributed.run on this node; rank 0 prints the line."""
    n_dev = visible_gpus()
    if n_dev < args.gpus:
        return refuse(args, n_dev)
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the communicator's rank count is in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_adaptive(args, H, ctx, y, points, nx, ny):
    """--adaptive TOL: K attempts of the adaptive BS3 loop (S12 with error
    partials, stage 3 with the error-norm epilogue, one 48-byte record read
    per attempt for the host PI controller, time_integration.hpp:301-344),
    wall-clock around one adaptive_solve call that stops on its step budget."""
    import torch
    tol = args.adaptive
    out = ctx.state()  # the result stays on the device (allocated outside the window)
    cfg = H.IntegratorConfig(abs_tol=tol, rel_tol=tol, max_steps=args.warmup)
    H.adaptive_solve(ctx, y, 0.0, 1e9, cfg, out=out)  # warm-up attempts (budget abort)
    cfg = H.IntegratorConfig(abs_tol=tol, rel_tol=tol, max_steps=args.steps)
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        clk.start()
        t0 = time.perf_counter()
        rec = H.adaptive_solve(ctx, y, 0.0, 1e9, cfg, out=out)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        clk.stop()
    attempts = rec.accepted + rec.rejected
    cfgd = workload_config(args, nx, ny, 1, "weak")
    cfgd["workload"] = cfgd["workload"].split(", fixed-step BS3")[0] + ", adaptive BS3"
    cfgd.update(integrator=f"adaptive BS3, abs_tol = rel_tol = {tol:g}, {attempts} attempts "
                           f"({rec.accepted} accepted, {rec.rejected} rejected), initial step estimated",
                l2="inputs > L2 (>= 2.7 GB per state, 126 MB L2); no flush needed")
    line = {"metric": METRIC, "value": 3 * points * attempts / el, "unit": UNIT, "n_gpus": 1,
            "steps": attempts, "warmup": args.warmup, "ms_per_step": 1e3 * el / max(attempts, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfgd, "timing": "wall clock around one adaptive_solve call "
            "(per-attempt host PI decisions included; its initial RHS and start-step estimate too)",
            "stop": rec.abort_reason, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--bc", default="periodic", choices=["periodic", "reflecting"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--config5", action="store_true", help="SURVEY config-5 shapes (16384 wide)")
    ap.add_argument("--n", type=int, default=0, help="nx (default 8192; 16384 for --config5 / strong N>1)")
    ap.add_argument("--rows", type=int, default=0, help="weak scaling: rows per rank (default nx; 4096 --config5)")
    ap.add_argument("--ny", type=int, default=0, help="strong scaling: global rows (default nx)")
    ap.add_argument("--sustained", type=int, default=300, help="steps of the sustained-rate run (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--rows-per-block", type=int, default=0)
    ap.add_argument("--fusion", type=int, default=-1, choices=[-1, 0, 3],
                    help="fixed-step kernel structure (0 per stage, 3 S12 + S3; -1 library default)")
    ap.add_argument("--adaptive", type=float, default=0.0, metavar="TOL",
                    help="N=1: time K adaptive BS3 attempts (abs = rel tolerance TOL, error norm on the device, "
                         "host PI controller) instead of fixed steps")
    ap.add_argument("--slab-ring", action="store_true",
                    help="N=1 only: run the P-rank slab code path as a 1-rank NCCL ring (halos to itself)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}\n")
        return 2
    import torch
    if torch.cuda.device_count() < max(world, local + 1):
        return refuse(args, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.slab_ring:
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2601_02540_b200 as H
    from paper_2601_02540_b200 import slab as S
    from paper_2601_02540_b200.workloads import bench_case

    nx, nyg, scaling = shapes(args, world)
    slabbed = world > 1 or args.slab_ring
    j0, j1 = S.partition(nyg, world)[rank]
    g, q, b, lam, dt, needs_aux = bench_case(args.bc, nx, nyg, rows=(j0, j1))
    phys = H.PhysSetup(9.81, lam, 1e-12, b.reshape(-1, nx))
    ctx = (S.make_slab_context(g, phys, rank, world, local, dist) if slabbed else
           H.make_rhs_context(g, phys, device=local))
    if args.rows_per_block:
        ctx.set_rows_per_block(args.rows_per_block)
    if args.fusion >= 0:
        ctx.fused_stages = args.fusion
    y = ctx.state(q)
    if needs_aux:  # w, eta of the reflecting workload (model.hpp:93-105, on the device)
        H.init_auxiliary(ctx, y)
        q = y.download().flat().copy()
    k1 = ctx.state()
    H.rhs(ctx, 0.0, y, k1)
    points = nx * ctx.ny_local

    if args.adaptive > 0:
        return run_adaptive(args, H, ctx, y, points, nx, nyg)

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed_steps(k, kernel_timing):
        """One hsgn_bs3_fixed_steps call of k steps (graphs built before the
        window); returns (done, max-over-ranks device ms, kernels, clocks)."""
        H.set_kernel_timing(ctx, kernel_timing)
        H.prepare_fixed_steps(ctx, y, k1, dt, k)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            clk.start()
            done, ms, kernels = H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, k)
            clk.stop()
        torch.cuda.synchronize()
        return done, max_over_ranks(ms), kernels, clk.summary()

    # warm-up (page-in, module load, first graph launches)
    H.set_kernel_timing(ctx, True)
    H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, args.warmup)
    # the timed region: K steps; CUDA event nodes around every kernel of the
    # captured graphs give the per-kernel durations of this very call
    done, ms_all, kernels, clocks = timed_steps(args.steps, True)
    s12_ms, s3_ms, kt_steps = H.kernel_times(ctx)
    value = 3 * points * world * args.steps / (ms_all * 1e-3)

    # roofline of the dominant kernel (S12): SURVEY 8(d) and own-byte views
    peak, peak_src = peaks()
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    fp64_peak = FP64_LANES_PER_SM * N_SM * sm_mhz * 1e-3  # G thread-instr/s at the sampled clock
    roofline = None
    if kt_steps and s12_ms > 0:
        kern = {}
        for name, t_ms in (("S12", s12_ms), ("S3", s3_ms)):
            sec = t_ms * 1e-3
            eq = BYTES_PER_POINT_STAGE * POINT_STAGES_PER_NODE[name] * points / sec / 1e9
            own = OWN_BYTES_PER_NODE[name] * points / sec / 1e9
            f64 = FP64_PER_NODE[name] * points / sec / 1e9
            kern[name] = {"ms": t_ms, "equiv_gbs": eq, "equiv_frac": eq / peak,
                          "own_bytes_per_node": OWN_BYTES_PER_NODE[name], "own_gbs": own, "own_frac": own / peak,
                          "fp64_instr_per_node": FP64_PER_NODE[name], "fp64_g_per_s": f64,
                          "fp64_frac": f64 / fp64_peak}
        traffic, tsrc = ncu_traffic("S12")
        dom = kern["S12"]
        roofline = {
            "bound": "hbm", "achieved": dom["equiv_gbs"], "peak": peak, "unit": "GB/s", "frac": dom["equiv_frac"],
            "traffic": traffic, "traffic_source": tsrc,
            "kernel": "sgn_s12_kernel (stages 1+2 of a BS3 step)",
            "definition": "SURVEY 8(d): 128 B per grid-point RK stage x 2 stages per node per S12 launch / mean "
                          "S12 launch time (CUDA event nodes inside the timed graphs)",
            "limiter": "FP64 dependency latency (own-byte HBM and FP64-pipe fractions below)",
            "own_bytes_frac": dom["own_frac"], "fp64_frac": dom["fp64_frac"],
            "fp64_peak_g_per_s": fp64_peak, "fp64_source": FP64_SOURCE, "peak_source": peak_src,
            "kernels": kern, "kernel_ms_steps_timed": kt_steps, "step_ms": ms_all / args.steps,
            "step_own_gbs": (OWN_BYTES_PER_NODE["S12"] + OWN_BYTES_PER_NODE["S3"]) * points
            / (ms_all / args.steps * 1e-3) / 1e9}

    # the same call without event nodes (the launch stream as shipped)
    done_b, ms_b, _, clocks_b = timed_steps(args.steps, False)
    plain = {"value": 3 * points * world * args.steps / (ms_b * 1e-3), "ms_per_step": ms_b / args.steps,
             "clocks": clocks_b}

    sustained = None
    if args.sustained > 0:
        done_s, ms_s, _, clocks_s = timed_steps(args.sustained, False)
        sustained = {"steps": args.sustained, "value": 3 * points * world * args.sustained / (ms_s * 1e-3),
                     "ms_per_step": ms_s / args.sustained, "clocks": clocks_s}

    # end-to-end through the public API with host buffers (pinned); at N > 1
    # every rank integrates its slab (halos and the step agreement over NCCL)
    e2e = None
    if not args.no_e2e:
        ny_l = ctx.ny_local
        host = torch.empty(q.size, dtype=torch.float64).pin_memory()
        host.numpy()[:] = q
        res_host = torch.empty(q.size, dtype=torch.float64).pin_memory()
        st_in = H.StateField((ny_l, nx), host.numpy())
        st_out = H.StateField((ny_l, nx), res_host.numpy())
        cfg = H.IntegratorConfig(fixed_dt=dt)
        dq0, out_state = ctx.state(), ctx.state()  # device buffers: allocated outside the window
        dq0.upload(st_in)
        H.adaptive_solve(ctx, dq0, 0.0, args.steps * dt, cfg, out=out_state)  # warm: builds its graphs
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dq0.upload(st_in)                                                  # H2D of the host state
        rec = H.adaptive_solve(ctx, dq0, 0.0, args.steps * dt, cfg, out=out_state)
        out_state.download(st_out)                                         # D2H of the result
        el = max_over_ranks(time.perf_counter() - t0)
        nbytes = 5 * points * 8 * world
        e2e = {"value": 3 * points * world * rec.accepted / el, "unit": UNIT,
               "h2d_bytes_per_step": nbytes / args.steps, "d2h_bytes_per_step": nbytes / args.steps,
               "api": "upload(pinned host q0) + adaptive_solve(fixed_dt, K steps, incl. initial RHS) + "
                      "download(q) -> pinned host" + (" per slab rank, max over ranks" if world > 1 else ""),
               "wall_s": el}
        dq0.free()
        out_state.free()

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(args.bc, nx, nyg)
        except Exception as ex:  # the baseline never gates the GPU number
            cb = {"value": None, "error": str(ex)}

    if rank == 0:
        cfg = workload_config(args, nx, nyg, world, scaling)
        cfg.update(l2="inputs > L2 (>= 2.7 GB per state, 126 MB L2); no flush needed",
                   rows_per_block=args.rows_per_block or "auto",
                   fixed_step_kernels="S12 + S3" if ctx.fused_stages == 3 else "one kernel per stage")
        if slabbed and world == 1:
            cfg["parallelism"] = "slab1 as a 1-rank NCCL ring (the P-rank code path)"
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_all / args.steps,
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": cfg,
                "hbm_gbs": roofline["step_own_gbs"] if roofline else None,
                "roofline": roofline, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": kernels,
                "clocks": clocks, "without_event_nodes": plain, "sustained": sustained, "steps_done": done}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
