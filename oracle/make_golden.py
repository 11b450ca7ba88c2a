#!/usr/bin/env python
"""Generate tests/golden/golden_r1.npz from the UNMODIFIED reference
(oracle/_ref/libhsgn_ref.so, built by `make -C oracle ref` from
/root/reference/proj/include).  TEST INFRASTRUCTURE ONLY.

The fixtures pin the C restatement (oracle/hsgn_oracle.c) on machines where
the reference tree is absent (the GPU box): tests/test_oracle.py checks the
restatement against them bit for bit, and tests/test_gpu_parity.py checks
the device path against the restatement.

Cases mirror the reference's own tests (file:line cited per case).
Run:  python oracle/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_lib import Oracle, Phys, default_cfg, make_grid, mms_exact_field, random_state  # noqa: E402


def grid_arr(g):
    return np.array([g.nx, g.ny, g.kind_x, g.kind_y, g.x_min, g.x_max, g.y_min, g.y_max], dtype=np.float64)


def sample(g, f):
    dx = (g.x_max - g.x_min) / (g.nx - 1 if g.kind_x else g.nx)
    dy = (g.y_max - g.y_min) / (g.ny - 1 if g.kind_y else g.ny)
    x = g.x_min + np.arange(g.nx) * dx
    y = g.y_min + np.arange(g.ny) * dy
    X, Y = np.meshgrid(x, y)
    return np.ascontiguousarray(np.broadcast_to(f(X, Y), X.shape)).ravel()


def main():
    ref = Oracle("ref")
    out = {}

    def rhs_case(name, g, lam, b, q, t=0.0, source=0, variant=0):
        st, o, _ = ref.rhs(g, Phys(9.81, lam, 1e-12), b, q, t=t, source_kind=source, variant=variant)
        assert st == 0, name
        out[f"rhs/{name}/grid"] = grid_arr(g)
        out[f"rhs/{name}/par"] = np.array([lam, t, source, variant], dtype=np.float64)
        out[f"rhs/{name}/b"] = b
        out[f"rhs/{name}/q"] = q
        out[f"rhs/{name}/out"] = o

    # test_rhs.cpp:84-94 (periodic, random state, seed 11 style)
    g = make_grid(24, 20)
    rhs_case("periodic_random", g, 500.0, sample(g, lambda x, y: 0.05 * np.sin(x + 2 * y)),
             random_state(24 * 20, 11))
    # test_rhs.cpp:95-105 (walls both directions)
    g = make_grid(24, 20, kind_x=1, kind_y=1)
    rhs_case("bounded_random", g, 500.0, sample(g, lambda x, y: 0.05 * np.cos(x - y)), random_state(24 * 20, 12))
    # test_rhs.cpp:108-127 mixed / lambda = 0 cases
    g = make_grid(20, 18, kind_x=1, kind_y=0)
    rhs_case("mixed_random", g, 500.0, sample(g, lambda x, y: 0.1 + 0.05 * np.sin(3 * x) * np.cos(y)),
             random_state(20 * 18, 22))
    g = make_grid(20, 18)
    rhs_case("lambda0_random", g, 0.0, sample(g, lambda x, y: 0.1 + 0.05 * np.sin(3 * x) * np.cos(y)),
             random_state(20 * 18, 21))
    rhs_case("shallow_water", g, 500.0, np.zeros(20 * 18), random_state(20 * 18, 31), variant=1)
    # manufactured state (SURVEY 8(d) benchmark input, small), with and without source
    g = make_grid(32, 32)
    q, b = mms_exact_field(g, 0.3)
    rhs_case("mms_state", g, 500.0, b, q)
    rhs_case("mms_source", g, 500.0, b, q, t=0.3, source=1)
    g = make_grid(33, 21, kind_x=1, kind_y=1)
    q, b = mms_exact_field(g, 0.3)
    rhs_case("mms_bounded", g, 500.0, b, q)
    # lake at rest over a bump (test_rhs.cpp:67-82), via init_auxiliary
    for kind in (0, 1):
        g = make_grid(33, 33, -5.0, 5.0, -5.0, 5.0, kind, kind)
        b = sample(g, lambda x, y: 0.1 * np.exp(-(x * x + y * y)))
        q = np.zeros(5 * 33 * 33)
        q[: 33 * 33] = 1.0 - b
        q = ref.init_auxiliary(g, b, q)
        out[f"init_aux/lake{kind}/q"] = q
        rhs_case(f"lake_at_rest{kind}", g, 500.0, b, q)

    # fixed-step BS3 (time_integration.hpp:209-350 with fixed_dt)
    for kind in (0, 1):
        g = make_grid(32, 24, kind_x=kind, kind_y=kind)
        q, b = mms_exact_field(g, 0.3)
        dt = 0.25 * (2.0 / 32) / 20.0
        T = 10 * dt + 0.4 * dt
        qf, rec = ref.solve(g, Phys(9.81, 500.0, 1e-12), b, q, 0.0, T, default_cfg(fixed_dt=dt))
        out[f"fixed/{kind}/grid"] = grid_arr(g)
        out[f"fixed/{kind}/b"] = b
        out[f"fixed/{kind}/q0"] = q
        out[f"fixed/{kind}/par"] = np.array([dt, T], dtype=np.float64)
        out[f"fixed/{kind}/q"] = qf
        out[f"fixed/{kind}/rec"] = np.array([rec.t, rec.accepted, rec.rejected, rec.rhs_evals,
                                             rec.rhs_evals_setup, rec.aborted], dtype=np.float64)
    # adaptive BS3 + PI controller, default tolerances (tolerance-level parity on device)
    g = make_grid(24, 24)
    q, b = mms_exact_field(g, 0.3)
    qf, rec = ref.solve(g, Phys(9.81, 500.0, 1e-12), b, q, 0.0, 0.01, default_cfg())
    out["adaptive/grid"] = grid_arr(g)
    out["adaptive/b"] = b
    out["adaptive/q0"] = q
    out["adaptive/q"] = qf
    out["adaptive/rec"] = np.array([rec.t, rec.accepted, rec.rejected, rec.rhs_evals, rec.rhs_evals_setup,
                                    rec.aborted], dtype=np.float64)

    # diagnostics (model.hpp:77-87, analysis.hpp:47-67)
    for name in ("periodic_random", "bounded_random", "mms_state"):
        gg = out[f"rhs/{name}/grid"]
        g = make_grid(int(gg[0]), int(gg[1]), gg[4], gg[5], gg[6], gg[7], int(gg[2]), int(gg[3]))
        lam = out[f"rhs/{name}/par"][0]
        ph = Phys(9.81, lam, 1e-12)
        q, b, qt = out[f"rhs/{name}/q"], out[f"rhs/{name}/b"], out[f"rhs/{name}/out"]
        out[f"diag/{name}"] = np.array([ref.total_mass(g, q), ref.total_energy(g, ph, b, q),
                                        ref.energy_rate(g, ph, b, q, qt)])

    # scenario inputs prepared by the reference itself (scenarios.hpp:55-78)
    for name, nx, ny, params in [("soliton", 64, 4, {}), ("gaussian_obstacle", 41, 21, {"bounded": 1.0}),
                                 ("manufactured", 16, 16, {}), ("lake_at_rest", 17, 17, {"bounded": 1.0})]:
        g, ph, b, q0, sk, t0, tf = ref.prepare(name, nx, ny, **params)
        out[f"scenario/{name}/grid"] = grid_arr(g)
        out[f"scenario/{name}/phys"] = np.array([ph.g, ph.lambda_, ph.h_floor, sk, t0, tf])
        out[f"scenario/{name}/b"] = b
        out[f"scenario/{name}/q0"] = q0

    # manufactured KATs evaluated by the reference (test_scenarios.cpp:92-136 points)
    pts = np.array([[0.3, 0.2, -0.4], [0.0, 0.3, 0.7], [0.0, 0.25, 0.25], [0.7, -0.9, 0.35]])
    out["mms/points"] = pts
    out["mms/state"] = np.array([ref.mms_state(*p) for p in pts])
    out["mms/state_dt"] = np.array([ref.mms_state_dt(*p) for p in pts])
    out["mms/source"] = np.array([ref.mms_source(*p) for p in pts])

    path = os.path.join(ROOT, "tests", "golden", "golden_r1.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
