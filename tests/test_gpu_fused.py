"""GPU: the fused stage-1 + stage-2 kernel (S12).

The fixed-step graphs run S12 + S3 per step (mode 3, the default) or one
kernel per stage (mode 0).  S12 must reproduce the unfused S1 and S2 bit
for bit, including at the tile seams (124 finished columns per CTA, two
halo columns each side), the CTA row seams (stage 1 re-runs one row above
and below each strip), the wrap / clamp rows and the edge / interior tile
split of grids with walls, and it must keep the reference's failure
semantics (which stage of which step failed, the abort reason, the ledger
and the last valid state).
"""
import numpy as np
import pytest

from oracle_lib import Oracle, Phys, default_cfg, make_grid as omake_grid, mms_exact_field

pytestmark = pytest.mark.gpu

import paper_2601_02540_b200 as H  # noqa: E402


@pytest.fixture(scope="module")
def orc():
    o = Oracle("orc")
    o.set_threads(8)
    return o


def _ctx(og, b, lam=500.0):
    g = H.make_grid(og.x_min, og.x_max, og.y_min, og.y_max, og.nx, og.ny, og.kind_x, og.kind_y)
    return g, H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(og.ny, og.nx)))


def _neq(a, b):
    return int(np.count_nonzero(np.asarray(a) != np.asarray(b)))


@pytest.mark.parametrize("nx,ny,kx,ky,rpb", [
    (64, 48, 0, 0, 0), (123, 9, 0, 0, 2), (124, 7, 0, 0, 3), (125, 11, 0, 0, 1), (126, 8, 1, 1, 4),
    (248, 6, 0, 1, 5), (249, 13, 1, 0, 0), (300, 21, 1, 1, 7), (4, 4, 0, 0, 0), (5, 6, 1, 1, 1),
    (128, 128, 0, 0, 0), (129, 65, 1, 1, 0), (256, 5, 0, 0, 2)])
def test_fused_fixed_steps_bitwise(orc, nx, ny, kx, ky, rpb):
    og = omake_grid(nx, ny, kind_x=kx, kind_y=ky)
    q, b = mms_exact_field(og, 0.3)
    dx = 2.0 / (nx - 1 if kx else nx)
    dt = 0.25 * dx / 20.0
    T = 9 * dt
    want, rec = orc.solve(og, Phys(9.81, 500.0, 1e-12), b, q, 0.0, T, default_cfg(fixed_dt=dt))
    g, ctx = _ctx(og, b)
    if rpb:
        ctx.set_rows_per_block(rpb)
    for mode in (0, 3):
        ctx.fused_stages = mode
        assert ctx.fused_stages == mode
        res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, T, H.IntegratorConfig(fixed_dt=dt))
        assert (res.accepted, res.rhs_evals, res.aborted) == (rec.accepted, rec.rhs_evals, bool(rec.aborted))
        assert _neq(res.q.flat(), want) == 0, f"mode {mode}"


def _drying_state(nx, ny, amp, U):
    x = -1 + np.arange(nx) * 2 / nx
    y = -1 + np.arange(ny) * 2 / ny
    X, Y = np.meshgrid(x, y)
    e = np.exp(-(X ** 2 + Y ** 2) / 0.05)
    h = 1 - amp * e
    return np.concatenate([h.ravel(), (U * X * e).ravel(), (U * Y * e).ravel(), np.zeros(nx * ny), h.ravel()])


# (amp, U, dt, h_floor): failures at stage 1, at stage 3, at the depth
# floor, and a floor hit on the first step
@pytest.mark.parametrize("amp,U,dt,floor", [(0.99, 10.0, 1e-3, 1e-12), (0.99, 30.0, 1e-3, 1e-12),
                                             (0.99, 10.0, 1e-3, 0.005), (0.999, 10.0, 1e-3, 0.005),
                                             (0.99, 10.0, 3e-3, 1e-12)])
@pytest.mark.parametrize("fused", [0, 3])
def test_fixed_step_failures_match_reference(orc, amp, U, dt, floor, fused):
    nx, ny = 64, 48
    og = omake_grid(nx, ny)
    q = _drying_state(nx, ny, amp, U)
    b = np.zeros(nx * ny)
    want, rec = orc.solve(og, Phys(9.81, 500.0, 1e-12), b, q, 0.0, 200 * dt,
                          default_cfg(fixed_dt=dt, h_floor=floor))
    assert rec.aborted
    g, ctx = _ctx(og, b)
    ctx.fused_stages = fused
    res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 200 * dt, H.IntegratorConfig(fixed_dt=dt, h_floor=floor))
    assert res.aborted
    assert res.abort_reason == rec.reason.decode()
    assert (res.accepted, res.rejected, res.rhs_evals) == (rec.accepted, rec.rejected, rec.rhs_evals)
    assert res.t == rec.t
    assert _neq(res.q.flat(), want) == 0


def test_fused_launch_count_and_profile():
    """Kernels per n-step graph chunk of a periodic grid: 3n per stage, 2n
    with S12 + S3; the other structures are rejected."""
    nx = ny = 256
    og = omake_grid(nx, ny)
    q, b = mms_exact_field(og, 0.3)
    g, ctx = _ctx(og, b)
    y = ctx.state(H.StateField(g, q))
    k1 = ctx.state()
    H.rhs(ctx, 0.0, y, k1)
    for mode, want in ((0, 3 * 64), (3, 2 * 64)):
        ctx.fused_stages = mode
        done, ms, kernels = H.bs3_fixed_steps(ctx, y, k1, 0.0, 1e-5, 64)
        assert done == 64 and kernels == want, mode
    for bad in (1, 2, 4):
        with pytest.raises(ValueError):
            ctx.fused_stages = bad


@pytest.mark.parametrize("kind", [0, 1])
def test_fused_structures_deterministic_under_repetition(kind):
    """Race detection by repetition (compute-sanitizer is unavailable on this
    pool): every kernel structure, 12 repetitions of 6 steps on a grid with
    partial tiles and short row strips, must give one bit pattern."""
    nx, ny = 1000, 300
    og = omake_grid(nx, ny, kind_x=kind, kind_y=kind)
    q, b = mms_exact_field(og, 0.3)
    g, ctx = _ctx(og, b)
    ctx.set_rows_per_block(5)
    dx = 2.0 / (nx - 1 if kind else nx)
    dt = 0.25 * dx / 20.0
    first = None
    for rep in range(12):
        for mode in (0, 3):
            ctx.fused_stages = mode
            res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 6 * dt, H.IntegratorConfig(fixed_dt=dt))
            flat = res.q.flat().copy()
            if first is None:
                first = flat
            assert _neq(flat, first) == 0, (rep, mode)


@pytest.mark.parametrize("kind,nx,ny", [(0, 96, 80), (1, 96, 80), (0, 400, 96), (1, 401, 131)])
def test_adaptive_attempts_fused_equal_unfused(kind, nx, ny):
    """Adaptive attempts run S12 (with the error partials) + S3 in mode 3:
    the error norms, hence the step sequence and the state, must equal the
    per-stage path bit for bit (the larger grids split into edge and
    interior launches, whose error partials share one array)."""
    og = omake_grid(nx, ny, kind_x=kind, kind_y=kind)
    q, b = mms_exact_field(og, 0.3)
    g, ctx = _ctx(og, b)
    res = {}
    for mode in (0, 3):
        ctx.fused_stages = mode
        r = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 0.02, H.IntegratorConfig(abs_tol=1e-8, rel_tol=1e-8))
        assert not r.aborted
        res[mode] = r
    assert (res[0].accepted, res[0].rejected, res[0].t) == (res[3].accepted, res[3].rejected, res[3].t)
    assert res[0].accepted > 3
    assert _neq(res[0].q.flat(), res[3].q.flat()) == 0


def test_fixed_step_errors_contract_at_third_order():
    """test_time_integration.cpp:72-86 on the device's own split-form RHS
    (the reference test integrates a scalar decay ODE through the generic
    callable, which the fused integrator does not take): a smooth periodic
    state integrated to T with dt and dt/2, errors against a dt/32 run; the
    ratio must be that of a third-order method, in (6.5, 9.5), for every
    field."""
    from paper_2601_02540_b200.workloads import mms_fields
    nx = ny = 48
    g, q, b = mms_fields(nx, ny, 0.3)
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(ny, nx)))
    T = 0.01

    def run(n):
        res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, T, H.IntegratorConfig(fixed_dt=T / n))
        assert not res.aborted and res.accepted == n
        return res.q.data

    ref = run(256)
    e1 = np.abs(run(8) - ref).reshape(5, -1).max(axis=1)
    e2 = np.abs(run(16) - ref).reshape(5, -1).max(axis=1)
    ratio = e1 / e2
    assert np.all((ratio > 6.5) & (ratio < 9.5)), ratio
