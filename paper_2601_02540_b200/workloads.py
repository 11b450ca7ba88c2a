"""Synthetic inputs of the BASELINE.json configurations (closed forms only).

The north-star benchmark input: periodic
[-1, 1]^2, bathymetry b = manufactured bathymetry (manufactured_generated.hpp
:11-15), state = manufactured exact solution at t = 0.3 (:18-38), g = 9.81,
lambda = 500, fixed dt = 0.25 dx / 20.  The closed form is restated here
(see DESIGN.md section 5); CPU and GPU arms receive the same arrays.
"""
from __future__ import annotations

import numpy as np

from .api import BoundaryKind, make_grid


def mms_fields(nx: int, ny: int, t: float, x_min=-1.0, x_max=1.0, y_min=-1.0, y_max=1.0,
               kind_x=BoundaryKind.periodic, kind_y=BoundaryKind.periodic, rows=None):
    """(grid, q (5*ny*nx), b (ny*nx)) of the manufactured solution at time t.
    rows=(j0, j1) samples only those global rows (a slab), q/b then hold
    j1-j0 rows."""
    g = make_grid(x_min, x_max, y_min, y_max, nx, ny, kind_x, kind_y)
    x = g.x(np.arange(nx))
    if rows is not None:
        y = g.y(np.arange(rows[0], rows[1]))
        ny = rows[1] - rows[0]
    else:
        y = g.y(np.arange(ny))
    tp, fp = 2 * np.pi, 4 * np.pi
    s1x, c1x, s2x, c2x = np.sin(tp * x), np.cos(tp * x), np.sin(fp * x), np.cos(fp * x)
    s1y, c1y, s2y, c2y = np.sin(tp * y), np.cos(tp * y), np.sin(fp * y), np.cos(fp * y)
    st, ct = np.sin(tp * t), np.cos(tp * t)
    q = np.empty((5, ny, nx))
    b = np.empty((ny, nx))
    chunk = max(1, (1 << 24) // nx)  # bounded temporaries for 8192^2
    for j0 in range(0, ny, chunk):
        sl = slice(j0, min(ny, j0 + chunk))
        S1y, C1y, S2y, C2y = s1y[sl, None], c1y[sl, None], s2y[sl, None], c2y[sl, None]
        bb = (2 / 25) * c1x * C1y + (1 / 25) * c2x * C2y
        bx = -(2 / 25) * tp * s1x * C1y - (1 / 25) * fp * s2x * C2y
        by = -(2 / 25) * tp * c1x * S1y - (1 / 25) * fp * c2x * S2y
        h = 2 + 0.5 * s1x * S1y * ct - bb
        u = 0.3 * s1x * st + 0 * S1y
        v = 0.3 * S1y * st + 0 * s1x
        ux = 0.3 * tp * c1x * st
        vy = 0.3 * tp * C1y * st
        b[sl] = bb
        q[0, sl] = h
        q[1, sl] = u
        q[2, sl] = v
        q[3, sl] = -h * (ux + vy) + 1.5 * (u * bx + v * by)
        q[4, sl] = h
    return g, q.reshape(-1), b.reshape(-1)


def benchmark_case(n: int = 8192):
    """Config 4 of BASELINE.json: (grid, q0, b, lambda, dt)."""
    g, q, b = mms_fields(n, n, 0.3)
    return g, q, b, 500.0, 0.25 * g.dx / 20.0


def bench_case(bc: str, nx: int, ny: int, rows=None):
    """The benchmark workloads (BASELINE configs 4 and 5) on an nx x ny grid,
    optionally only global rows (j0, j1) of it (a slab's share).

    * ``periodic``: the config-4 input -- manufactured bathymetry and state at
      t = 0.3 -- on [-1, 1] x [-1, -1 + 2 ny / nx] (dx == dy, so every nx with
      nx | 2^k keeps the common-factor stencil; the state has period 1 in y,
      so a 2P-long domain is the same smooth periodic input);
    * ``reflecting``: ``gaussian_obstacle(bounded)`` (scenarios.hpp:356-383) --
      walls on all four sides, SBP closures and SAT -- sampled by the
      scenario library; w and eta come from the device init_auxiliary
      (``needs_aux``).
    Returns (grid, q, b, lambda, dt, needs_aux)."""
    if bc == "periodic":
        g, q, b = mms_fields(nx, ny, 0.3, y_max=-1.0 + 2.0 * ny / nx, rows=rows)
        return g, q, b, 500.0, 0.25 * g.dx / 20.0, False
    if bc == "reflecting":
        from .scenarios import make_scenario, sample_rows
        spec = make_scenario("gaussian_obstacle", {"bounded": 1.0})
        g = spec.grid(nx, ny)
        j0, j1 = rows if rows is not None else (0, ny)
        b, q = sample_rows(spec, nx, ny, j0, j1)
        return g, q, b, spec.lambda_, 0.25 * min(g.dx, g.dy) / 20.0, True
    raise ValueError(f"unknown boundary workload {bc!r}")
