"""GPU: the device path against the UNMODIFIED reference (oracle/_ref, the
reference headers compiled in place) at the BASELINE configurations' own
sizes, and the reference's acceptance gates that need a device tendency.

* config 4: 10 fixed BS3 steps of the 8192^2 benchmark workload, full-grid
  IEEE-== comparison (5 x 67,108,864 values; the reference runs on the host
  cores, ~40 s);
* config 1: the first 1,000 fixed steps of the solitary wave on 256 x 256
  (lambda = 30000, dt = 1.5e-3) from the reference's own prepare_run state;
* config 3: the reflecting basin (gaussian_obstacle, bounded: SBP closures
  and SAT on all four walls) on 512 x 512, 200 fixed steps, bitwise;
* acceptance c2 (acceptance_main.cpp:88-127): the 300 random 32 x 32 states
  of the gate (the reference's own mt19937 stream), periodic / reflecting /
  lambda = 0: device RHS bitwise equal to the reference's and the
  semidiscrete energy rate <= 1e-11 E;
* acceptance c4 (acceptance_main.cpp:148-160): lake at rest 65 x 65, both
  kinds: max |tendency| <= 1e-12 g.
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle_lib import Oracle, Phys, default_cfg, make_grid as omake, ref_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")]

import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200.workloads import benchmark_case  # noqa: E402


@pytest.fixture(scope="module")
def ref():
    o = Oracle("ref")
    o.set_threads(os.cpu_count() or 8)
    return o


def _neq(a, b):
    return int(np.count_nonzero(np.asarray(a) != np.asarray(b)))


def _dev_grid(g):
    return H.make_grid(g.x_min, g.x_max, g.y_min, g.y_max, g.nx, g.ny, g.kind_x, g.kind_y)


def test_config4_full_size_10_steps_bitwise(ref):
    n, steps = 8192, 10
    g, q, b, lam, dt = benchmark_case(n)
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(n, n)), device=0)
    dev = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, steps * dt, H.IntegratorConfig(fixed_dt=dt))
    got = dev.q.flat().copy()
    del dev
    ctx.close()
    want, rr = ref.solve(omake(n, n), Phys(9.81, lam, 1e-12), b, q, 0.0, steps * dt, default_cfg(fixed_dt=dt))
    assert rr.accepted == steps and not rr.aborted
    assert _neq(got, want) == 0


def test_config1_soliton_1000_steps_bitwise(ref):
    from paper_2601_02540_b200.scenarios import make_scenario, prepare_run
    g, ph, b, q0, sk, t0, tf = ref.prepare("soliton", 256, 256)
    dt, steps = 1.5e-3, 1000
    run = prepare_run(make_scenario("soliton"), 256, 256, device=0)
    assert _neq(run.q0.download().flat(), q0) == 0, "initial states differ"
    dev = H.adaptive_solve(run.ctx, run.q0, t0, t0 + steps * dt, H.IntegratorConfig(fixed_dt=dt))
    want, rr = ref.solve(g, ph, b, q0, t0, t0 + steps * dt, default_cfg(fixed_dt=dt))
    assert (dev.accepted, dev.t) == (rr.accepted, rr.t)
    assert _neq(dev.q.flat(), want) == 0


@pytest.mark.parametrize("rpb", [0, 7])
def test_config3_reflecting_basin_512_bitwise(ref, rpb):
    g, ph, b, q0, sk, t0, tf = ref.prepare("gaussian_obstacle", 512, 512, bounded=1.0)
    assert g.kind_x == 1 and g.kind_y == 1
    grid = _dev_grid(g)
    ctx = H.make_rhs_context(grid, H.PhysSetup(ph.g, ph.lambda_, ph.h_floor, b.reshape(512, 512)))
    if rpb:
        ctx.set_rows_per_block(rpb)
    dt = 0.25 * min(grid.dx, grid.dy) / 20.0
    steps = 200
    dev = H.adaptive_solve(ctx, H.StateField(grid, q0), t0, t0 + steps * dt, H.IntegratorConfig(fixed_dt=dt))
    want, rr = ref.solve(g, ph, b, q0, t0, t0 + steps * dt, default_cfg(fixed_dt=dt))
    assert (dev.accepted, dev.t) == (rr.accepted, rr.t)
    assert _neq(dev.q.flat(), want) == 0
    # mass conserved to round-off over the run (c3 analogue)
    m0 = H.total_mass(ctx, H.StateField(grid, q0))
    m1 = H.total_mass(ctx, dev.q)
    assert abs(m1 - m0) <= 1e-12 * abs(m0)


def test_acceptance_c2_energy_rate_random_states(ref):
    n_setups, trials, n = 3, 100, 32 * 32
    states = np.empty(n_setups * trials * 5 * n)
    ref.lib.ref_c2_states.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double)]
    ref.lib.ref_c2_states(n_setups, trials, states.ctypes.data_as(C.POINTER(C.c_double)))
    states = states.reshape(n_setups, trials, 5 * n)
    worst = 0.0
    for s, (kind, lam) in enumerate(((0, 500.0), (1, 500.0), (0, 0.0))):
        og = omake(32, 32, kind_x=kind, kind_y=kind)
        grid = _dev_grid(og)
        x, y = grid.x(np.arange(32)), grid.y(np.arange(32))
        X, Y = np.meshgrid(x, y)
        b = (0.02 + 0.08 * np.exp(-2.0 * (X * X + Y * Y))).ravel()
        ph = Phys(9.81, lam, 1e-12)
        ctx = H.make_rhs_context(grid, H.PhysSetup(9.81, lam, 1e-12, b.reshape(32, 32)))
        for t in range(trials):
            q = states[s, t]
            qt = H.StateField(grid)
            H.rhs(ctx, 0.0, H.StateField(grid, q), qt)
            st, want, _ = ref.rhs(og, ph, b, q)
            assert st == 0
            assert _neq(qt.flat(), want) == 0, (s, t)
            dq, dqt = ctx.state(H.StateField(grid, q)), ctx.state(qt)
            e = H.total_energy(ctx, dq)
            rate = H.energy_rate(ctx, dq, dqt)
            worst = max(worst, abs(rate) / abs(e))
            dq.free()
            dqt.free()
        ctx.close()
    assert worst <= 1e-11, worst


@pytest.mark.parametrize("bounded", [0.0, 1.0])
def test_acceptance_c4_lake_at_rest(ref, bounded):
    g, ph, b, q0, sk, t0, tf = ref.prepare("lake_at_rest", 65, 65, bounded=bounded)
    grid = _dev_grid(g)
    ctx = H.make_rhs_context(grid, H.PhysSetup(ph.g, ph.lambda_, ph.h_floor, b.reshape(65, 65)))
    qt = H.StateField(grid)
    H.rhs(ctx, 0.0, H.StateField(grid, q0), qt)
    st, want, _ = ref.rhs(g, ph, b, q0)
    assert _neq(qt.flat(), want) == 0
    assert np.max(np.abs(qt.flat())) <= 1e-12 * 9.81 * 1.0
