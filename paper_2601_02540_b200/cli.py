"""Command-line front end of the reference (cli.hpp:1-304, tools/hsgn_main.cpp)
on the device path:

    python -m paper_2601_02540_b200.cli run      --config run.cfg [--output DIR] [--threads N]
    python -m paper_2601_02540_b200.cli converge --config study.cfg [--output DIR]
    python -m paper_2601_02540_b200.cli bench    [--config bench.cfg] [--output DIR]

Same configuration files (config.py), scenarios (scenarios.py), output files
(gauges.csv, snapshot_t*.csv, conservation.csv, cross_section.csv,
convergence.csv, bench.csv -- byte-compatible %.17g writers) and run_meta.json
keys as the reference; exit codes 0 ok, 1 solver abort / failed rung,
2 configuration error.  The integration runs on the B200 through the fused
kernels (adaptive_solve) with the on-device RunRecorder; `threads` is parsed
and recorded (it sets the reference's host thread count) but the device path
does not use host threads.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from typing import List, Optional, TextIO

import numpy as np

from . import api as H
from .config import ConfigError, RunConfig, apply_thread_env, parse_config_file
from .recorder import RunRecorder, fmt17, fmt_short, write_cross_section_csv
from .scenarios import FIELD_NAMES, ScenarioSpec, exact_state, make_scenario, prepare_run, study_case


def _boundary_name(k) -> str:
    return "periodic" if int(k) == 0 else "reflecting"


def _num(v):
    """nlohmann::json stores non-finite doubles as null."""
    return v if (not isinstance(v, float) or math.isfinite(v)) else None


def _integrator_json(c: H.IntegratorConfig) -> dict:
    """cli.hpp:26-37"""
    return {"abs_tol": c.abs_tol, "rel_tol": c.rel_tol, "dt_initial": c.dt_initial,
            "dt_max": c.dt_max if math.isfinite(c.dt_max) else "inf", "fixed_dt": c.fixed_dt,
            "max_steps": int(c.max_steps), "safety": c.safety, "growth_cap": c.growth_cap,
            "shrink_floor": c.shrink_floor}


def _base_meta(command: str, cfg: RunConfig, spec: ScenarioSpec, grid) -> dict:
    """cli.hpp:39-60 (plus the device the run used)."""
    return {"command": command,
            "scenario": {"name": spec.name, "parameters": dict(cfg.scenario_params)},
            "grid": {"nx": grid.nx, "ny": grid.ny, "dx": grid.dx, "dy": grid.dy, "x_min": grid.x_min,
                     "x_max": grid.x_max, "y_min": grid.y_min, "y_max": grid.y_max,
                     "boundary_x": _boundary_name(grid.kind_x), "boundary_y": _boundary_name(grid.kind_y)},
            "physics": {"g": spec.g, "lambda": spec.lambda_},
            "threads": cfg.threads,
            "device": "B200 (sm_100a), " + H.N.lib().hsgn_build_info().decode()}


def _write_json(path: str, j: dict) -> None:
    """cli.hpp:62-67 (nlohmann dump(2): sorted keys, 2-space indent)."""
    def clean(o):
        if isinstance(o, dict):
            return {k: clean(v) for k, v in o.items()}
        if isinstance(o, (list, tuple)):
            return [clean(v) for v in o]
        return _num(o)
    try:
        with open(path, "w") as fh:
            fh.write(json.dumps(clean(j), indent=2, sort_keys=True) + "\n")
    except OSError:
        raise RuntimeError(f"cannot write '{path}'") from None


def _apply_overrides(cfg: RunConfig, spec: ScenarioSpec):
    """cli.hpp:70-82"""
    nx = cfg.nx if cfg.nx > 0 else spec.nx_default
    ny = cfg.ny if cfg.ny > 0 else spec.ny_default
    if not math.isnan(cfg.t0):
        spec.t0 = cfg.t0
    if not math.isnan(cfg.t_final):
        spec.t_final = cfg.t_final
    if cfg.gauges_set:
        spec.gauges = list(cfg.gauges)
    if cfg.snapshots_set:
        spec.snapshot_times = list(cfg.snapshot_times)
    return nx, ny


def cmd_run(cfg: RunConfig, log: TextIO = sys.stdout, device: int = -1) -> int:
    """cli.hpp:88-157: one scenario with gauges / snapshots / conservation
    records; 0 on a completed run, 1 when the solver aborts."""
    spec = make_scenario(cfg.scenario, cfg.scenario_params)
    nx, ny = _apply_overrides(cfg, spec)
    os.makedirs(cfg.output_dir, exist_ok=True)
    run = prepare_run(spec, nx, ny, device)
    ctx = run.ctx
    log.write(f"run: scenario {spec.name} on {nx}x{ny} grid, t in [{fmt_short(spec.t0)}, "
              f"{fmt_short(spec.t_final)}]\n")
    rec = RunRecorder(ctx, cfg.output_dir, spec.gauges, spec.snapshot_times, cfg.conservation_stride)
    mass0 = H.total_mass(ctx, run.q0)
    energy0 = H.total_energy(ctx, run.q0)
    wall0 = time.perf_counter()
    sol = H.adaptive_solve(ctx, run.q0, spec.t0, spec.t_final, cfg.integrator, recorder=rec)
    wall = time.perf_counter() - wall0
    rec.flush()
    if cfg.cross_section_set:
        write_cross_section_csv(cfg.output_dir + "/cross_section.csv", run.grid, sol.q.flat(), run.b,
                                cfg.cross_section_y)
    mass1 = H.total_mass(ctx, sol.device_q)
    energy1 = H.total_energy(ctx, sol.device_q)

    meta = _base_meta("run", cfg, spec, run.grid)
    meta["time"] = {"t0": spec.t0, "t_final": spec.t_final, "t_reached": sol.t}
    meta["integrator"] = _integrator_json(cfg.integrator)
    meta["steps"] = {"accepted": sol.accepted, "rejected": sol.rejected, "rhs_evals": sol.rhs_evals,
                     "rhs_evals_setup": sol.rhs_evals_setup}
    meta["conservation"] = {"mass_initial": mass0, "mass_final": mass1, "mass_drift_rel": (mass1 - mass0) / mass0,
                            "energy_initial": energy0, "energy_final": energy1,
                            "energy_drift_rel": (energy1 - energy0) / energy0}
    meta["snapshots"] = [{"target": s.target, "actual": s.actual, "file": os.path.basename(s.path)}
                         for s in rec.snapshots()]
    meta["output"] = {"directory": cfg.output_dir, "conservation_stride": cfg.conservation_stride}
    meta["wall_seconds"] = wall
    meta["status"] = "aborted" if sol.aborted else "ok"
    if sol.aborted:
        meta["abort_reason"] = sol.abort_reason
    _write_json(cfg.output_dir + "/run_meta.json", meta)
    rec.close()
    log.write(f"run: {'ABORTED: ' + sol.abort_reason if sol.aborted else 'completed'} at t = {fmt_short(sol.t)} "
              f"({sol.accepted} accepted, {sol.rejected} rejected, {sol.rhs_evals} tendency evaluations, "
              f"{fmt_short(wall)} s)\n"
              f"run: relative mass drift {fmt_short((mass1 - mass0) / mass0)}, relative energy drift "
              f"{fmt_short((energy1 - energy0) / energy0)}\n")
    sol.device_q.free()
    run.q0.free()
    ctx.close()
    return 1 if sol.aborted else 0


class ConvergenceTable:
    """analysis.hpp ConvergenceTable: per rung nx, dx, errors, rates, status."""

    def __init__(self):
        self.variables: List[str] = []
        self.resolution: List[int] = []
        self.dx: List[float] = []
        self.errors: List[List[float]] = []
        self.rates: List[List[float]] = []
        self.status: List[str] = []


def run_convergence_study(spec: ScenarioSpec, resolutions: List[int], icfg: H.IntegratorConfig, ny_fixed: int = 0,
                          device: int = -1) -> ConvergenceTable:
    """scenarios.hpp:535-592 on the device: each rung integrated with the
    fused pipeline, errors as SBP-norm discrete L2 distances to the exact
    state (analysis.hpp:15-25), rates by eoc (analysis.hpp:29-39)."""
    if len(resolutions) < 2:
        raise ValueError("run_convergence_study: need at least 2 resolutions")
    for r in range(1, len(resolutions)):
        if resolutions[r] <= resolutions[r - 1]:
            raise ValueError("run_convergence_study: resolutions must be strictly increasing")
    nan = math.nan
    t = ConvergenceTable()
    for r, n in enumerate(resolutions):
        ny = ny_fixed if ny_fixed > 0 else n
        case = study_case(spec, n, ny, device)
        ctx = case.ctx
        if not t.variables:
            t.variables = list(spec.exact_vars)
        rec = H.adaptive_solve(ctx, case.q0, spec.t0, spec.t_final, icfg)
        t.resolution.append(n)
        t.dx.append(case.grid.dx)
        if rec.aborted:
            t.errors.append([nan] * len(t.variables))
            t.rates.append([nan] * len(t.variables))
            t.status.append("failed: " + rec.abort_reason)
            rec.device_q.free()
            case.q0.free()
            ctx.close()
            continue
        ref = H.StateField(case.grid, exact_state(spec, n, ny, rec.t))
        errs = [H.discrete_l2_error(ctx, rec.device_q, ref, FIELD_NAMES.index(v)) for v in t.variables]
        t.errors.append(errs)
        rates = [nan] * len(errs)
        if r > 0 and t.status[-1] == "ok":
            rates = [H.eoc(t.errors[r - 1][v], errs[v], t.dx[r - 1], t.dx[r]) for v in range(len(errs))]
        t.rates.append(rates)
        t.status.append("ok")
        rec.device_q.free()
        case.q0.free()
        ctx.close()
    return t


def write_convergence_csv(path: str, t: ConvergenceTable) -> None:
    """io.hpp:79-93"""
    with open(path, "w") as out:
        out.write("nx,dx" + "".join(f",err_{v},eoc_{v}" for v in t.variables) + ",status\n")
        for r in range(len(t.resolution)):
            out.write(f"{t.resolution[r]},{fmt17(t.dx[r])}")
            for v in range(len(t.variables)):
                out.write(f",{fmt17(t.errors[r][v])},{fmt17(t.rates[r][v])}")
            out.write(f",{t.status[r]}\n")


def cmd_converge(cfg: RunConfig, log: TextIO = sys.stdout, device: int = -1) -> int:
    """cli.hpp:161-216: refinement study; 0 when every rung completed."""
    spec = make_scenario(cfg.scenario, cfg.scenario_params)
    _apply_overrides(cfg, spec)
    if not spec.has_exact:
        raise ValueError(f"cmd_converge: scenario '{spec.name}' has no exact solution to converge against")
    if len(cfg.resolutions) < 2:
        raise ValueError("cmd_converge: [converge] resolutions needs >= 2 entries")
    os.makedirs(cfg.output_dir, exist_ok=True)
    icfg = H.IntegratorConfig(**vars(cfg.integrator))
    if not cfg.tolerances_set:
        icfg.abs_tol = 1e-10  # spatial error must dominate
        icfg.rel_tol = 1e-10
    log.write(f"converge: scenario {spec.name}, resolutions" + "".join(f" {n}" for n in cfg.resolutions)
              + f", tolerances {fmt_short(icfg.abs_tol)}\n")
    wall0 = time.perf_counter()
    table = run_convergence_study(spec, cfg.resolutions, icfg, cfg.converge_ny, device)
    wall = time.perf_counter() - wall0
    write_convergence_csv(cfg.output_dir + "/convergence.csv", table)
    all_ok = True
    for r in range(len(table.resolution)):
        line = f"converge: nx = {table.resolution[r]}"
        for v, name in enumerate(table.variables):
            line += f"  err_{name} = {fmt_short(table.errors[r][v])} (eoc {fmt_short(table.rates[r][v])})"
        log.write(line + f"  [{table.status[r]}]\n")
        all_ok = all_ok and table.status[r] == "ok"
    n0 = cfg.resolutions[0]
    grid0 = spec.grid(n0, cfg.converge_ny if cfg.converge_ny > 0 else n0)
    meta = _base_meta("converge", cfg, spec, grid0)
    meta["integrator"] = _integrator_json(icfg)
    meta["resolutions"] = list(cfg.resolutions)
    meta["status"] = "ok" if all_ok else "failed"
    meta["row_status"] = list(table.status)
    meta["wall_seconds"] = wall
    _write_json(cfg.output_dir + "/run_meta.json", meta)
    return 0 if all_ok else 1


def cmd_bench(cfg: RunConfig, log: TextIO = sys.stdout, device: int = -1) -> int:
    """cli.hpp:221-302: tendency-evaluation throughput over a resolution
    ladder (seconds per device rhs(), host-timed around the synchronous call
    like the reference's steady_clock); bench.csv + run_meta.json."""
    c = RunConfig(**vars(cfg))
    if not c.scenario:
        c.scenario = "still_water"
    for n in c.bench_resolutions:
        if n < 4:
            raise ValueError(f"cmd_bench: resolution {n} is below the 4-node minimum")
    if not c.bench_resolutions:
        raise ValueError("cmd_bench: empty resolution ladder")
    if c.bench_repetitions < 1 or c.bench_warmups < 0:
        raise ValueError("cmd_bench: need repetitions >= 1 and warmups >= 0")
    spec = make_scenario(c.scenario, c.scenario_params)
    os.makedirs(c.output_dir, exist_ok=True)
    rungs = []
    for n in c.bench_resolutions:
        run = prepare_run(spec, n, n, device)
        out = run.ctx.state()
        for _ in range(c.bench_warmups):
            H.rhs(run.ctx, spec.t0, run.q0, out)
        secs = []
        for _ in range(c.bench_repetitions):
            a = time.perf_counter()
            H.rhs(run.ctx, spec.t0, run.q0, out)
            secs.append(time.perf_counter() - a)
        secs.sort()
        k = c.bench_repetitions
        med = secs[k // 2] if k % 2 == 1 else 0.5 * (secs[k // 2 - 1] + secs[k // 2])
        rungs.append((n, med, secs[0]))
        log.write(f"bench: {n}x{n}  median {fmt_short(med * 1e3)} ms  min {fmt_short(secs[0] * 1e3)} ms per "
                  f"evaluation\n")
        out.free()
        run.q0.free()
        run.ctx.close()
    with open(c.output_dir + "/bench.csv", "w") as out:
        out.write("nx,ny,n_total,seconds_per_rhs,seconds_per_rhs_min,threads\n")
        for n, med, mn in rungs:
            out.write(f"{n},{n},{n * n},{fmt17(med)},{fmt17(mn)},{c.threads}\n")
    n0 = c.bench_resolutions[0]
    meta = _base_meta("bench", c, spec, spec.grid(n0, n0))
    meta["repetitions"] = c.bench_repetitions
    meta["warmups"] = c.bench_warmups
    meta["rungs"] = [{"nx": n, "ny": n, "n_total": n * n, "seconds_per_rhs": med, "seconds_per_rhs_min": mn}
                     for n, med, mn in rungs]
    meta["status"] = "ok"
    _write_json(c.output_dir + "/run_meta.json", meta)
    return 0


def _resolve(args) -> RunConfig:
    """hsgn_main.cpp CommonArgs::resolve: --threads over the config key over
    THREADS; --output over the config directory."""
    cfg = parse_config_file(args.config) if args.config else RunConfig()
    apply_thread_env(cfg)
    if args.threads and args.threads > 0:
        cfg.threads = args.threads
    if args.output:
        cfg.output_dir = args.output
    return cfg


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="hsgn", description="Dispersive shallow-water solver: split-form finite "
                                 "differences for the hyperbolic Serre-Green-Naghdi equations (B200 device path)")
    sub = ap.add_subparsers(dest="command", required=True)
    for name, required, hlp in (("run", True, "Integrate one scenario and record results"),
                                ("converge", True, "Grid-refinement study against an exact solution"),
                                ("bench", False, "Tendency-evaluation throughput over a resolution ladder")):
        p = sub.add_parser(name, help=hlp)
        p.add_argument("--config", required=required, help="Path to the key = value configuration file")
        p.add_argument("--output", help="Output directory (overrides the config file)")
        p.add_argument("--threads", type=int, default=0, help="Worker thread count (overrides config and THREADS)")
    args = ap.parse_args(argv)
    try:
        cfg = _resolve(args)
        return {"run": cmd_run, "converge": cmd_converge, "bench": cmd_bench}[args.command](cfg)
    except (ConfigError, ValueError, RuntimeError, OSError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
