#!/usr/bin/env python
"""Benchmark of the fused fp64 SGN split-form BS3 stage pipeline on B200.

Metric (BASELINE.json): grid-point RK-stage updates per second on an 8192^2
fp64 grid (config 4: periodic [-1,1]^2, manufactured bathymetry and state at
t = 0.3, lambda = 500, fixed dt = 0.25 dx / 20), plus achieved HBM GB/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 8192]

* ``value``   : point-stage updates/s, device time (CUDA events on the
                library stream) of K graph-captured fused steps, inputs
                resident in HBM; every state is 2.7 GB (> 126 MB L2), so no
                L2 flush is needed between steps.
* ``e2e``     : the same metric through the public API with HOST buffers:
                one ``adaptive_solve`` call (fixed dt, K steps) from a pinned
                host state to a host result, H2D + D2H inside the timed region.
* ``roofline``: the dominant kernel of the steady-state step (S2 or the
                fused S3+S1 kernel S31, DESIGN.md sections 2b, 7), algorithmic
                bytes per launch (168 / 128 B per node) / its mean launch time.
* ``cpu_baseline``: the reference CPU path (oracle/_ref, or the C oracle port)
                on this host's cores on a bounded sample.
Multi-GPU (torchrun): weak scaling, every rank owns an 8192-row slab of a
(8192 x 8192*N) periodic grid; halo rows via NCCL.  ``--impl reference``
runs the reference CPU implementation only on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_NODE = {"S1": 128, "S2": 168, "S3": 88, "S31": 128, "STEP": 168, "S12": 128}
BYTES_PER_POINT_STAGE = 128  # unfused step: 384 B per node / 3 stages
# FP64 instructions (DADD + DMUL + DFMA) per node of each kernel, from the ncu
# SASS mixes in profiles/ (r1_sass_mix_stage_kernels.txt, r1f_sass_mix_s31.txt,
# r1k_sass_mix_s12.txt, r1k_sass_mix_s3.txt): the compute roofline of the FP64-issue-bound kernels
FP64_PER_NODE = {"S1": 199.5, "S2": 228.8, "S3": 189.1, "S31": 397.3, "S12": 437.5}
FP64_LANES_PER_SM, N_SM = 64, 148


def step_bytes_per_node(mode: int, chunk: int) -> float:
    """Algorithmic HBM bytes per node per step of the fixed-step pipeline:
    mode 0 S1 + S2 + S3 = 384; mode 1 chunks of n steps S1 + n S2 +
    (n-1) S31 + S3 = 296 n + 88; mode 2 one whole-step kernel = 168;
    mode 3 S12 + S3 = 128 + 88 = 216."""
    if mode == 0:
        return 384.0
    if mode == 1:
        return (296.0 * chunk + 88.0) / chunk
    return 168.0 if mode == 2 else 216.0
METRIC = "grid-point RK-stage updates/sec on 8192² fp64 grid; achieved HBM GB/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region:
    sampling starts before and stops after it, and only the samples stamped
    inside [start(), stop()] (the timed call) enter the summary."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period_ms=20):
        self.index = index
        self.period_ms = period_ms
        self.samples = []
        self._p = None
        self._t0 = self._t1 = None

    # cumulative microseconds each limiter held the clocks down: the delta
    # over the timed call catches a limiter between two instantaneous samples
    CQ = ("clocks_event_reasons_counters.sw_power_cap,clocks_event_reasons_counters.sw_thermal_slowdown,"
          "clocks_event_reasons_counters.hw_thermal_slowdown,clocks_event_reasons_counters.hw_power_brake_slowdown")
    CNAMES = ("sw_power_cap", "sw_thermal_slowdown", "hw_thermal_slowdown", "hw_slowdown")

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
            if len(parts) >= 7:
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
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = {names[k] for s in self.samples for k in range(4) if "Active" in s[2 + k] and "Not" not in s[2 + k]}
        held = {}
        c0, c1 = getattr(self, "_c0", None), getattr(self, "_c1", None)
        if c0 and c1 and len(c0) == len(c1) == 4:
            for k, nm in enumerate(self.CNAMES):
                if c1[k] > c0[k]:
                    reasons.add(nm)
                    held[nm + "_ms"] = (c1[k] - c0[k]) / 1e3
        reasons = sorted(reasons)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "limiter_ms": held, "samples": len(self.samples),
                "window": "timed call only" if getattr(self, "windowed", False) else "whole sampler run"}


class CpuReference:
    """The reference CPU implementation of the path on this host's cores:
    oracle/_ref (the unmodified reference headers compiled in place; OpenMP)
    when it was built, else the C oracle port.  A "step" is one fixed-step
    BS3 step (time_integration.hpp:262-345: 3 RHS + stage axpys + min-h) of
    an n^2 sample of the benchmark workload (same closed-form input)."""

    def __init__(self, n: int):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_lib import PD, Oracle, Phys, default_cfg, make_grid as omake, ref_available
        from paper_2601_02540_b200.workloads import mms_fields
        self.kind = "reference" if ref_available() else "port"
        self.orc = Oracle("ref" if self.kind == "reference" else "orc")
        self.cores = os.cpu_count() or 1
        self.orc.set_threads(self.cores)
        self.n = n
        g, self.q, self.b = mms_fields(n, n, 0.3)
        self.og = omake(n, n)
        self.dt = 0.25 * g.dx / 20.0
        self.ph = Phys(9.81, 500.0, 1e-12)
        self.cfg = default_cfg
        self._pd = PD

    def steps(self, k: int) -> float:
        """Wall seconds of k fixed steps, minus the initial tendency the
        solve evaluates first (timed separately as one RHS)."""
        t0 = time.perf_counter()
        _, rec = self.orc.solve(self.og, self.ph, self.b, self.q, 0.0, k * self.dt, self.cfg(fixed_dt=self.dt))
        el = time.perf_counter() - t0
        assert rec.accepted == k and not rec.aborted
        return el * (3 * k) / (3 * k + 1)  # drop the k1 = f(y0) evaluation's share

    def describe(self, k, seconds):
        return {"value": 3 * k * self.n * self.n / seconds, "unit": "point-stage updates/s", "cores": self.cores,
                "kind": self.kind,
                "sample": f"{self.n}x{self.n} slice of the config-4 workload (periodic, manufactured state "
                          f"t=0.3, lambda=500), {k} fixed BS3 steps via the reference adaptive_solve(fixed_dt), "
                          f"{seconds:.2f} s wall on {self.cores} threads"}


def cpu_baseline(n_sample: int = 2048, steps: int = 12):
    ref = CpuReference(n_sample)
    ref.steps(1)  # warm-up: page-in, OpenMP pool
    return ref.describe(steps, ref.steps(steps))


def workload_config(n: int, world: int) -> dict:
    """The workload both arms report (BASELINE config 4; weak scaling stacks
    8192-row slabs)."""
    nyg = n * world
    return {"workload": f"config 4: {n}x{nyg} periodic, manufactured bathymetry + state "
                        f"(t=0.3), lambda=500, fixed-step BS3 dt=0.25dx/20",
            "grid": f"{n}x{nyg}", "points": n * nyg, "parallelism": f"slab{world}"}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation, timed per
    step on this host's cores (rank 0 only under torchrun)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ref = CpuReference(args.ref_n)
    ref.steps(max(1, args.warmup))  # warm-up steps (page-in, OpenMP pool, workspace first touch)
    total = ref.steps(args.steps)   # K steps in one solve, as the reference integrates
    cb = ref.describe(args.steps, total)
    v = cb["value"]
    line = {"metric": METRIC, "value": v, "unit": "point-stage updates/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            # the same workload as the device arm; each step runs on the bounded
            # sample cpu_baseline.sample states (host cores, OpenMP)
            "config": dict(workload_config(args.n, args.gpus), parallelism="cpu-openmp",
                           sample=f"{args.ref_n}x{args.ref_n} slice per step"),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "point-stage updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--ref-n", type=int, default=2048)
    ap.add_argument("--ref-steps", type=int, default=12)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--rows-per-block", type=int, default=0)
    ap.add_argument("--fusion", type=int, default=-1, choices=[-1, 0, 1, 2, 3],
                    help="fixed-step kernel structure (0 per stage, 1 S31, 2 whole step, 3 S12 + S3; "
                         "-1 library default)")
    ap.add_argument("--slab-ring", action="store_true",
                    help="N=1 only: run the P-rank slab code path as a 1-rank NCCL ring (halos to itself)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
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
    from paper_2601_02540_b200.workloads import mms_fields

    n = args.n
    nyg = n * world
    slabbed = world > 1 or args.slab_ring
    g, q, b = mms_fields(n, nyg, 0.3) if not slabbed else S.slab_fields(n, nyg, 0.3, rank, world)
    dt = 0.25 * (2.0 / n) / 20.0
    phys = H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(-1, n))
    if not slabbed:
        ctx = H.make_rhs_context(g, phys, device=local)
    else:
        ctx = S.make_slab_context(g, phys, rank, world, local, dist)
    if args.rows_per_block:
        ctx.set_rows_per_block(args.rows_per_block)
    if args.fusion >= 0:
        ctx.fused_stages = args.fusion
    mode = ctx.fused_stages if not slabbed else (3 if ctx.fused_stages == 3 else 0)  # slabs: S12 + S3 or per stage
    y = ctx.state(q)
    k1 = ctx.state()
    H.rhs(ctx, 0.0, y, k1)
    points = n * ctx.ny_local

    # warm-up; the CUDA graphs of the timed K-step call are built here too
    # (capture + instantiation is one-time host work, not a step)
    H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, args.warmup)
    H.prepare_fixed_steps(ctx, dt, args.steps)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        clk.start()
        done, ms, kernels = H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, args.steps)
        clk.stop()
    torch.cuda.synchronize()
    ms_all = ms
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_all = float(t.item())
    value = 3 * points * world * args.steps / (ms_all * 1e-3)

    # per-kernel times for the roofline (same stream, CUDA events)
    ms3 = (H.api.N.D * 3)()
    H.api._check(ctx, H.api.N.lib().hsgn_profile_stages(ctx._h, y._h, k1._h, dt, 3, ms3), "profile")
    ms3 = list(ms3)
    names = ["S1", "S2", "S3"]
    if mode:  # steady-state step: S2 + S31 (mode 1), STEP (mode 2), S12 + S3 (mode 3)
        mf = H.api.N.D(0.0)
        H.api._check(ctx, H.api.N.lib().hsgn_profile_fused(ctx._h, y._h, k1._h, dt, 3, H.api.C.byref(mf)),
                     "profile_fused")
        ms3.append(mf.value)
        names.append({1: "S31", 2: "STEP", 3: "S12"}[mode])
    cand = {0: [0, 1, 2], 1: [1, 3], 2: [3], 3: [2, 3]}[mode]
    dom = max(cand, key=lambda k: ms3[k])
    peak, peak_kind = peaks()
    achieved = BYTES_PER_NODE[names[dom]] * points / (ms3[dom] * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(names[dom])
    fp64 = None
    if names[dom] in FP64_PER_NODE:
        sm_mhz = clk.summary().get("sm_mhz") or 1965.0
        got = FP64_PER_NODE[names[dom]] * points / (ms3[dom] * 1e-3) / 1e9
        top = FP64_LANES_PER_SM * N_SM * sm_mhz * 1e-3
        fp64 = {"unit": "G FP64 thread-instr/s", "instr_per_node": FP64_PER_NODE[names[dom]], "achieved": got,
                "peak": top, "frac": got / top, "peak_basis": f"{FP64_LANES_PER_SM} lanes x {N_SM} SMs x sm_mhz"}
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "fp64": fp64,
                "traffic": traffic,
                "kernel": {"S31": "sgn_s31_kernel", "STEP": "sgn_step_kernel", "S12": "sgn_s12_kernel"}.get(
                    names[dom], f"sgn_stage_kernel<{names[dom]}>"),
                "fixed_step_kernels": ["per stage", "S2 + S31", "whole step", "S12 + S3"][mode],
                "bytes_per_node": BYTES_PER_NODE[names[dom]], "peak_source": peak_kind,
                "stage_ms": {names[k]: ms3[k] for k in range(len(names))},
                "step_bytes_per_node": step_bytes_per_node(mode, min(64, args.steps)),
                # updates/s x 128 B (the unfused compulsory traffic per
                # point-stage) against the HBM peak; fusion removes traffic, so this
                # equivalent-bandwidth fraction exceeds the fused kernels' own
                "equiv_unfused": {"bytes_per_point_stage": BYTES_PER_POINT_STAGE,
                                  "achieved": value * BYTES_PER_POINT_STAGE / 1e9,
                                  "frac": value * BYTES_PER_POINT_STAGE / 1e9 / peak},
                "step_gbs": step_bytes_per_node(mode, min(64, args.steps)) * points / (ms / args.steps * 1e-3) / 1e9}

    # end-to-end through the public API with host buffers (pinned); at N > 1
    # every rank integrates its slab (halos and the step agreement over NCCL)
    e2e = None
    if not args.no_e2e:
        ny_l = ctx.ny_local
        host = torch.empty(q.size, dtype=torch.float64).pin_memory()
        host.numpy()[:] = q
        res_host = torch.empty(q.size, dtype=torch.float64).pin_memory()
        st_in = H.StateField((ny_l, n), host.numpy())
        cfg = H.IntegratorConfig(fixed_dt=dt)
        out_state = ctx.state()
        # warm: the same call, so the timed one reuses its CUDA graphs
        H.adaptive_solve(ctx, st_in, 0.0, args.steps * dt, cfg, out=out_state)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        dq0 = ctx.state(st_in)                        # H2D of the host state
        rec = H.adaptive_solve(ctx, dq0, 0.0, args.steps * dt, cfg, out=out_state)
        out_state.download(H.StateField((ny_l, n), res_host.numpy()))  # D2H of the result
        el = time.perf_counter() - t0
        if dist:
            t = torch.tensor([el], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        nbytes = 5 * points * 8 * world
        e2e = {"value": 3 * points * world * rec.accepted / el, "unit": "point-stage updates/s",
               "h2d_bytes_per_step": nbytes / args.steps, "d2h_bytes_per_step": nbytes / args.steps,
               "api": "adaptive_solve(host q0 -> host q, fixed_dt, K steps) incl. initial RHS"
                      + (" per slab rank, max over ranks" if world > 1 else ""),
               "wall_s": el}
        dq0.free()
        out_state.free()

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(args.ref_n, args.ref_steps)
        except Exception as ex:  # the baseline never gates the GPU number
            cb = {"value": None, "error": str(ex)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "point-stage updates/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_all / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": dict(workload_config(n, world),
                               l2="inputs > L2 (2.7 GB per state); no flush needed",
                               rows_per_block=args.rows_per_block or "auto",
                               **({"parallelism": "slab1 as a 1-rank NCCL ring (the P-rank code path)"}
                                  if slabbed and world == 1 else {})),
                "hbm_gbs": roofline["step_gbs"], "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
                "gpu_launches": kernels, "clocks": clk.summary(), "steps_done": done}
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
