"""Scenario registry and run preparation of the reference CLI front end
(scenarios.hpp:18-707), over the native registry in hsgn_scenarios.cpp.

    spec = make_scenario("soliton", {"amplitude": 0.1})   # make_scenario, :598-698
    run = prepare_run(spec, nx, ny)                         # prepare_run, :55-78
    run.ctx, run.grid, run.q0 (DeviceState)

The initial b, h, u, v are evaluated on the host by the native registry
(bit-identical to the reference's closed forms, same libm); w and eta come
from the device init_auxiliary, the manufactured forcing is the context's
device source term (hsgn_set_source).  Nothing here integrates on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .api import BoundaryKind, DeviceState, Grid2D, PhysSetup, RhsContext, init_auxiliary, make_grid

FIELD_NAMES = ("h", "u", "v", "w", "eta")


@dataclass
class ScenarioSpec:
    """scenarios.hpp:21-46 (the closed forms live in the native registry)."""
    name: str
    x_min: float
    x_max: float
    y_min: float
    y_max: float
    nx_default: int
    ny_default: int
    kind_x: BoundaryKind
    kind_y: BoundaryKind
    g: float
    lambda_: float
    t0: float
    t_final: float
    has_source: bool
    has_exact: bool
    exact_vars: List[str]
    gauges: List[Tuple[float, float]] = field(default_factory=list)
    snapshot_times: List[float] = field(default_factory=list)
    _c: Optional[N.hsgn_scenario] = None

    def grid(self, nx: int, ny: int) -> Grid2D:
        return make_grid(self.x_min, self.x_max, self.y_min, self.y_max, nx, ny, self.kind_x, self.kind_y)


def scenario_names() -> List[str]:
    """scenarios.hpp:700-705"""
    L = N.lib()
    return [L.hsgn_scenario_name(k).decode() for k in range(L.hsgn_scenario_count())]


def make_scenario(name: str, params: Optional[Dict[str, float]] = None) -> ScenarioSpec:
    """make_scenario (scenarios.hpp:598-698): unknown names or parameters
    raise ValueError with the reference message (std::invalid_argument)."""
    params = dict(params or {})
    keys = (C.c_char_p * max(1, len(params)))(*[k.encode() for k in params])
    vals = np.array([float(v) for v in params.values()] or [0.0], dtype=np.float64)
    out = N.hsgn_scenario()
    err = C.create_string_buffer(256)
    st = N.lib().hsgn_scenario_make(name.encode(), keys, vals.ctypes.data_as(N.PD), len(params), C.byref(out), err,
                                    256)
    if st:
        raise ValueError(err.value.decode())
    d = out.domain
    return ScenarioSpec(
        name=out.name.decode(), x_min=d.x_min, x_max=d.x_max, y_min=d.y_min, y_max=d.y_max, nx_default=d.nx,
        ny_default=d.ny, kind_x=BoundaryKind(d.kind_x), kind_y=BoundaryKind(d.kind_y), g=out.g,
        lambda_=out.lambda_, t0=out.t0, t_final=out.t_final, has_source=bool(out.has_source),
        has_exact=bool(out.has_exact), exact_vars=[FIELD_NAMES[out.exact_vars[k]] for k in range(out.n_exact_vars)],
        gauges=[(out.gauges[k][0], out.gauges[k][1]) for k in range(out.n_gauges)],
        snapshot_times=[out.snapshot_times[k] for k in range(out.n_snapshots)], _c=out)


def sample_initial(spec: ScenarioSpec, nx: int, ny: int) -> Tuple[np.ndarray, np.ndarray]:
    """(b (ny*nx), q (5*ny*nx) with h, u, v sampled and w = eta = 0)."""
    spec.grid(nx, ny)  # make_grid validation and messages
    b = np.empty(nx * ny)
    q = np.empty(5 * nx * ny)
    st = N.lib().hsgn_scenario_sample(C.byref(spec._c), nx, ny, b.ctypes.data_as(N.PD), q.ctypes.data_as(N.PD))
    if st:
        raise ValueError(f"hsgn_scenario_sample failed ({st})")
    return b, q


def sample_rows(spec: ScenarioSpec, nx: int, ny: int, j0: int, j1: int) -> Tuple[np.ndarray, np.ndarray]:
    """sample_initial restricted to global rows [j0, j1) (a slab): b
    ((j1-j0)*nx), q (5*(j1-j0)*nx) with w = eta = 0."""
    spec.grid(nx, ny)
    m = (j1 - j0) * nx
    b = np.empty(m)
    q = np.empty(5 * m)
    st = N.lib().hsgn_scenario_sample_rows(C.byref(spec._c), nx, ny, j0, j1, b.ctypes.data_as(N.PD),
                                           q.ctypes.data_as(N.PD))
    if st:
        raise ValueError(f"hsgn_scenario_sample_rows failed ({st})")
    return b, q


def evaluate(spec: ScenarioSpec, x: float, y: float):
    """The spec's closed forms at one point: (b, h0, u0, v0)(x, y)
    (spec.bathymetry / h0 / u0 / v0, scenarios.hpp:31-34)."""
    out = np.empty(4)
    st = N.lib().hsgn_scenario_eval(C.byref(spec._c), float(x), float(y), out.ctypes.data_as(N.PD))
    if st:
        raise ValueError(f"hsgn_scenario_eval failed ({st})")
    return tuple(float(v) for v in out)


def exact_state(spec: ScenarioSpec, nx: int, ny: int, t: float) -> np.ndarray:
    """The scenario's exact solution at time t (5*ny*nx), scenarios.hpp:155-170, 200-214."""
    if not spec.has_exact:
        raise ValueError(f"scenario '{spec.name}' has no exact solution")
    q = np.empty(5 * nx * ny)
    st = N.lib().hsgn_scenario_exact(C.byref(spec._c), nx, ny, float(t), q.ctypes.data_as(N.PD))
    if st:
        raise ValueError(f"hsgn_scenario_exact failed ({st})")
    return q


@dataclass
class PreparedRun:
    """scenarios.hpp:49-53: grid, context (with the source hook) and q0 on the device."""
    grid: Grid2D
    ctx: RhsContext
    q0: DeviceState
    b: np.ndarray


def prepare_run(spec: ScenarioSpec, nx: int = 0, ny: int = 0, device: int = -1) -> PreparedRun:
    """prepare_run (scenarios.hpp:55-78): sample b, h, u, v; create the
    context (manufactured forcing as the device source term); w and eta from
    the device init_auxiliary."""
    nx = nx or spec.nx_default
    ny = ny or spec.ny_default
    grid = spec.grid(nx, ny)
    b, q = sample_initial(spec, nx, ny)
    ctx = RhsContext(grid, PhysSetup(spec.g, spec.lambda_, 1e-12, b.reshape(ny, nx)), device=device)
    if spec.has_source:
        ctx.source = "manufactured"
    q0 = ctx.state(q)
    init_auxiliary(ctx, q0)
    return PreparedRun(grid, ctx, q0, b)


def study_case(spec: ScenarioSpec, nx: int, ny: int, device: int = -1) -> PreparedRun:
    """study_case_from (scenarios.hpp:515-533)."""
    if not spec.has_exact:
        raise ValueError(f"study_case_from: scenario '{spec.name}' has no exact solution")
    return prepare_run(spec, nx, ny, device)


__all__ = ["ScenarioSpec", "PreparedRun", "scenario_names", "make_scenario", "sample_initial", "sample_rows",
           "exact_state", "evaluate",
           "prepare_run", "study_case", "FIELD_NAMES"]
