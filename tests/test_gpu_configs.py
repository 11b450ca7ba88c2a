"""GPU tests of the BASELINE.json configurations (parity + physics gates).

config 1  soliton, flat bottom, periodic, 256 x 256, fixed-step BS3
          -> state bitwise equal to the oracle after 300 steps (config 1 recipe,
             SURVEY.md section 8(d))
config 2  manufactured solution with variable bathymetry, periodic
          -> device sources within 1e-12 of the oracle; observed order of
             convergence in [1.8, 2.2] (acceptance_main.cpp:182-203)
config 3  reflecting basin with variable bathymetry (SBP closures + SAT)
          -> mass drift <= 1e-12 relative over a long run; semidiscrete
             energy rate <= 1e-11 E at every recorded step (acceptance c2/c3)
config 4  8192^2 periodic benchmark input
          -> bitwise parity on random windows (the tendency of a node only
             depends on its 3x3 neighbourhood), size-independent properties
             (mass rate, energy rate, determinism) on the full grid
"""
import numpy as np
import pytest

from oracle_lib import Oracle, Phys, default_cfg, make_grid as omake_grid, mms_exact_field

pytestmark = pytest.mark.gpu

import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200.workloads import mms_fields  # noqa: E402


@pytest.fixture(scope="module")
def orc():
    o = Oracle("orc")
    o.set_threads(8)
    return o


def soliton_state(nx, ny):
    """soliton_1d defaults (scenarios.hpp:123-172): h_inf=1, A=0.2, g=9.81,
    lambda=30000, [-30,30]^2, along x; eta = h, w from init_auxiliary."""
    h_inf, A, g = 1.0, 0.2, 9.81
    eps = A / h_inf
    kappa = np.sqrt(3 * eps / (4 * h_inf * h_inf * (1 + eps)))
    c = np.sqrt(g * h_inf * (1 + eps))
    grid = H.make_grid(-30.0, 30.0, -30.0, 30.0, nx, ny)
    x = grid.x(np.arange(nx))
    h = h_inf + A / np.cosh(kappa * x) ** 2
    u = c * (1 - h_inf / h)
    q = np.zeros((5, ny, nx))
    q[0] = h
    q[1] = u
    return grid, q.reshape(-1), np.zeros(nx * ny)


def test_config1_soliton_bitwise(orc):
    nx = ny = 256
    grid, q, b = soliton_state(nx, ny)
    og = omake_grid(nx, ny, -30.0, 30.0, -30.0, 30.0)
    ph = Phys(9.81, 30000.0, 1e-12)
    q = orc.init_auxiliary(og, b, q)
    dt = 1.5e-3
    T = 300 * dt
    want, rec = orc.solve(og, ph, b, q, 0.0, T, default_cfg(fixed_dt=dt))
    ctx = H.make_rhs_context(grid, H.PhysSetup(9.81, 30000.0, 1e-12, b.reshape(ny, nx)))
    qs = H.StateField(grid, q)
    res = H.adaptive_solve(ctx, qs, 0.0, T, H.IntegratorConfig(fixed_dt=dt))
    assert not res.aborted and res.accepted == rec.accepted and res.t == rec.t
    assert np.count_nonzero(res.q.flat() != want) == 0


def test_config2_manufactured_sources_and_order(orc):
    # device sources vs oracle on one rung
    g, q, b = mms_fields(128, 128, 0.3)
    og = omake_grid(128, 128)
    st, want, _ = orc.rhs(og, Phys(9.81, 500.0, 1e-12), b, q, t=0.3, source_kind=1)
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(128, 128)))
    ctx.source = "manufactured"
    out = H.StateField(g)
    H.rhs(ctx, 0.3, H.StateField(g, q), out)
    assert np.max(np.abs(out.flat() - want)) <= 1e-12 * np.max(np.abs(want))
    # convergence: fixed dt at the CFL limit, temporal error O(dt^3) << spatial O(dx^2)
    errs, dxs = [], []
    T = 0.25
    for n in (64, 128, 256):
        g, q0, b = mms_fields(n, n, 0.0)
        ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(n, n)))
        ctx.source = "manufactured"
        dt = T / int(np.ceil(T / (0.25 * g.dx / 20.0)))
        res = H.adaptive_solve(ctx, H.StateField(g, q0), 0.0, T, H.IntegratorConfig(fixed_dt=dt))
        assert not res.aborted and res.t == pytest.approx(T)
        _, qe, _ = mms_fields(n, n, res.t)
        exact = H.StateField(g, qe)
        errs.append([H.discrete_l2_error(ctx, res.q, exact, f) for f in range(5)])
        dxs.append(g.dx)
    for f in range(5):
        rate = H.eoc(errs[1][f], errs[2][f], dxs[1], dxs[2])
        assert 1.8 <= rate <= 2.2, (f, rate, errs)


def test_config3_reflecting_basin_conservation():
    """Gaussian bump under a solitary front, walls on all sides (gaussian_obstacle
    bounded, scenarios.hpp:356-383), 512^2 slice of the 4096^2 config."""
    n = 512
    g = H.make_grid(-5.0, 35.0, -10.0, 10.0, n, n, H.BoundaryKind.bounded, H.BoundaryKind.bounded)
    b = g.sample(lambda x, y: 0.1 * np.exp(-0.5 * (x * x + y * y)))
    h_inf, A = 0.2, 0.0365
    eps = A / h_inf
    kappa = np.sqrt(3 * eps / (4 * h_inf * h_inf * (1 + eps)))
    c = np.sqrt(9.81 * h_inf * (1 + eps))
    q = H.StateField(g)
    q.h[:] = g.sample(lambda x, y: h_inf + A / np.cosh(kappa * (x + 3.0)) ** 2) - b
    q.u[:] = g.sample(lambda x, y: c * (1 - h_inf / (h_inf + A / np.cosh(kappa * (x + 3.0)) ** 2)))
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, b))
    H.init_auxiliary(ctx, q)
    m0 = H.total_mass(ctx, q)
    worst_rate = [0.0]

    def obs(t, qd, qtd):
        e = H.total_energy(ctx, qd)
        r = H.energy_rate(ctx, qd, qtd)
        worst_rate[0] = max(worst_rate[0], abs(r) / abs(e))

    dt = 0.5 * min(g.dx, g.dy) / (np.sqrt(9.81 * 0.3) + np.sqrt(500.0 / 3) + 1.0)
    res = H.adaptive_solve(ctx, q, 0.0, 400 * dt, H.IntegratorConfig(fixed_dt=dt), on_accept=obs)
    assert not res.aborted and res.accepted == 400
    m1 = H.total_mass(ctx, res.q)
    assert abs(m1 - m0) <= 1e-12 * abs(m0)
    assert worst_rate[0] <= 1e-11


@pytest.mark.slow
def test_config4_windows_bitwise_and_properties(orc):
    n = 8192
    g, q, b = mms_fields(n, n, 0.3)
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(n, n)))
    assert ctx.stencil_kind == 2
    dq = ctx.state(q)
    dout = ctx.state()
    H.rhs(ctx, 0.0, dq, dout)
    out = dout.download().data
    Q = q.reshape(5, n, n)
    B = b.reshape(n, n)
    rng = np.random.default_rng(5)
    import ctypes as C
    from oracle_lib import PD, Grid
    fn = orc.lib.orc_rhs_dxdy
    fn.restype = C.c_int
    fn.argtypes = [C.POINTER(Grid), C.c_double, C.c_double, C.POINTER(Phys), PD, C.c_int, C.c_double, PD, PD]
    w = 48
    corners = [(0, 0), (n - w, n - w), (0, n - w)] + [tuple(rng.integers(0, n - w, 2)) for _ in range(5)]
    for (j0, i0) in corners:
        rows = np.arange(j0 - 1, j0 + w + 1) % n
        cols = np.arange(i0 - 1, i0 + w + 1) % n
        qw = np.ascontiguousarray(Q[:, rows][:, :, cols]).ravel()
        bw = np.ascontiguousarray(B[rows][:, cols]).ravel()
        og = omake_grid(w + 2, w + 2)
        ow = np.empty_like(qw)
        assert fn(C.byref(og), g.dx, g.dy, C.byref(Phys(9.81, 500.0, 1e-12)), bw.ctypes.data_as(PD), 0, 0.0,
                  qw.ctypes.data_as(PD), ow.ctypes.data_as(PD)) == 0
        want = ow.reshape(5, w + 2, w + 2)[:, 1:-1, 1:-1]
        got = out[:, j0:j0 + w, i0:i0 + w]
        assert np.count_nonzero(got != want) == 0, (j0, i0)
    # size-independent properties on the full grid
    assert abs(H.mass_weighted_sum(ctx, dout, 0)) <= 1e-12 * H.total_mass(ctx, dq)   # 1^T M h_t
    e = H.total_energy(ctx, dq)
    r = H.energy_rate(ctx, dq, dout)
    assert abs(r) <= 1e-11 * abs(e)
    dout2 = ctx.state()
    H.rhs(ctx, 0.0, dq, dout2)
    assert np.array_equal(dout2.download().data, out)   # deterministic, bit for bit


def test_fixed_step_failure_semantics(orc):
    """Depth loss inside a graph chunk: same abort reason, time and state as
    the reference (time_integration.hpp:291-296)."""
    n = 64
    g, q, b = mms_fields(n, n, 0.3)
    og = omake_grid(n, n)
    dt = 0.02  # far beyond CFL: the state blows up and loses depth after a few steps
    want, rec = orc.solve(og, Phys(9.81, 500.0, 1e-12), b, q, 0.0, 200 * dt, default_cfg(fixed_dt=dt))
    assert rec.aborted
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(n, n)))
    res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 200 * dt, H.IntegratorConfig(fixed_dt=dt))
    assert res.aborted
    assert res.abort_reason == rec.reason.decode()
    assert (res.t, res.accepted, res.rhs_evals) == (rec.t, rec.accepted, rec.rhs_evals)
    assert np.count_nonzero(res.q.flat() != want) == 0


def test_adaptive_solve_matches_reference_closely(orc):
    """Adaptive BS3 + PI controller (time_integration.hpp:301-344): the only
    divergence source is the order of the error-norm sum."""
    for kx in (0, 1):
        og = omake_grid(48, 48, kind_x=kx, kind_y=kx)
        q, b = mms_exact_field(og, 0.3)
        want, rec = orc.solve(og, Phys(9.81, 500.0, 1e-12), b, q, 0.0, 0.02, default_cfg())
        g = H.make_grid(-1.0, 1.0, -1.0, 1.0, 48, 48, kx, kx)
        ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(48, 48)))
        res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 0.02, H.IntegratorConfig())
        assert not res.aborted and res.t == rec.t
        assert abs(res.accepted - rec.accepted) <= 1 and res.rhs_evals_setup == rec.rhs_evals_setup
        assert np.max(np.abs(res.q.flat() - want)) <= 1e-9 * np.max(np.abs(want))


def test_config3_full_4096_long_time(tmp_path):
    """BASELINE config 3 at its stated size: the reflecting basin
    (gaussian_obstacle, walls on all four sides, variable bathymetry) on a
    4096 x 4096 grid, 3000 fixed steps through the CLI path (scenario
    registry + on-device recorder, a conservation row every 250 steps).
    Mass is a linear invariant of the scheme: drift <= 1e-12 relative over
    the whole run.  The semidiscrete energy rate is round-off: |dE/dt| <=
    1e-11 E at every record.  The fully discrete energy drift is the BS3
    time-integration error (small, not round-off)."""
    from paper_2601_02540_b200 import cli
    from paper_2601_02540_b200.config import RunConfig
    spec_dt = 0.5 * (20.0 / 4095) / (np.sqrt(9.81 * 0.3) + np.sqrt(500.0 / 3) + 1.0)
    cfg = RunConfig(scenario="gaussian_obstacle", scenario_params={"bounded": 1.0}, nx=4096, ny=4096,
                    t_final=3000 * spec_dt, output_dir=str(tmp_path / "basin"), conservation_stride=250,
                    gauges_set=True, gauges=[(0.0, 0.0)], snapshots_set=True, snapshot_times=[])
    cfg.integrator.fixed_dt = spec_dt
    import io
    log = io.StringIO()
    assert cli.cmd_run(cfg, log) == 0, log.getvalue()
    import json
    meta = json.load(open(tmp_path / "basin" / "run_meta.json"))
    assert meta["status"] == "ok" and meta["grid"]["nx"] == 4096 and meta["grid"]["boundary_y"] == "reflecting"
    assert meta["steps"]["accepted"] >= 2999
    assert abs(meta["conservation"]["mass_drift_rel"]) <= 1e-12
    assert abs(meta["conservation"]["energy_drift_rel"]) <= 1e-6
    rows = [ln.split(",") for ln in open(tmp_path / "basin" / "conservation.csv").read().splitlines()[1:]]
    cons = np.array([[float(x) for x in r] for r in rows])
    assert len(cons) >= 12
    print("config3 4096^2:", meta["steps"], meta["conservation"], "max |rate|/E",
          float(np.max(np.abs(cons[:, 3]) / np.abs(cons[:, 2]))), "wall", meta["wall_seconds"])
    assert np.all(np.abs(cons[:, 1] - cons[0, 1]) <= 1e-12 * abs(cons[0, 1]))
    assert np.all(np.abs(cons[:, 3]) <= 1e-11 * np.abs(cons[:, 2]))
