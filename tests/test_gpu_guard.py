"""GPU: the magnitude guard of the fast tendency association and the
two-pass tiles, and manufactured sources in the fused
S12 + S3 pipeline.

* states with subnormal-range velocities (a wavefront entering water at
  rest), on periodic power-of-two grids (stencil kind 2: the common factor)
  and on walls (kind 0): RHS and fixed BS3 steps bit-identical to the oracle,
  in both kernel structures and with tiles that switch between the fast and
  the literal pass from step to step (the per-tile hints);
* tiny nonzero bathymetry forces the literal association everywhere under
  the common factor (host-checked): still bit-identical;
* sources in S12 + S3 (fixed and adaptive) agree with the per-stage
  structure and with the oracle to the source tolerance (device sin / cos
  are not correctly rounded).
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


def _neq(a, b):
    return int(np.count_nonzero(np.asarray(a) != np.asarray(b)))


def _ctx(og, b, lam=500.0):
    g = H.make_grid(og.x_min, og.x_max, og.y_min, og.y_max, og.nx, og.ny, og.kind_x, og.kind_y)
    return g, H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(og.ny, og.nx)))


def _front_state(og, tiny_b=False):
    """Water at rest (h = eta = 1, u = v = w = 0) with a bump on the left:
    velocities and w decay through every magnitude to the subnormals (and
    to exact zeros) across the grid -- the regime of the guard."""
    nx, ny = og.nx, og.ny
    x = og.x_min + np.arange(nx) * (og.x_max - og.x_min) / (nx - 1 if og.kind_x else nx)
    y = og.y_min + np.arange(ny) * (og.y_max - og.y_min) / (ny - 1 if og.kind_y else ny)
    X, Y = np.meshgrid(x, y)
    r2 = (X + 0.6) ** 2 + Y ** 2
    h = 1.0 + 0.1 * np.exp(-r2 / 0.01)
    u = 0.3 * np.exp(-r2 / 0.002)  # ~exp(-400 r^2): subnormal far away, exact zero beyond
    v = -0.2 * np.exp(-r2 / 0.002) * Y
    w = 1e-3 * np.exp(-r2 / 0.0015) * X
    b = 0.05 * np.exp(-((X - 0.3) ** 2 + Y ** 2) / 0.05) if not tiny_b else 0.05 * np.exp(-750.0 * (X + 1.0))
    q = np.concatenate([h.ravel(), u.ravel(), v.ravel(), w.ravel(), h.ravel()])
    return q, b.ravel()


def test_front_state_has_tiny_values():
    og = omake_grid(128, 96)
    q, b = _front_state(og)
    u = q[128 * 96:2 * 128 * 96]
    nz = np.abs(u[u != 0])
    assert (nz < 2.0 ** -120).any() and (nz < 2.2e-308).any() and (u == 0).any()


@pytest.mark.parametrize("nx,ny,kx,ky,rpb", [(128, 96, 0, 0, 0), (256, 64, 0, 0, 7), (129, 97, 1, 1, 0),
                                            (200, 80, 1, 1, 5)])
def test_rhs_bitwise_with_subnormal_front(orc, nx, ny, kx, ky, rpb):
    og = omake_grid(nx, ny, kind_x=kx, kind_y=ky)
    q, b = _front_state(og)
    st, want, _ = orc.rhs(og, Phys(9.81, 500.0, 1e-12), b, q)
    assert st == 0
    g, ctx = _ctx(og, b)
    if rpb:
        ctx.set_rows_per_block(rpb)
    out = H.StateField(g)
    H.rhs(ctx, 0.0, H.StateField(g, q), out)
    assert _neq(out.flat(), want) == 0


@pytest.mark.parametrize("nx,ny,kx,ky", [(128, 96, 0, 0), (129, 97, 1, 1), (256, 128, 0, 0)])
def test_fixed_steps_bitwise_with_moving_front(orc, nx, ny, kx, ky):
    """40 steps: the front crosses tile boundaries, so tiles switch between
    the fast and the literal pass (and their hints) along the run."""
    og = omake_grid(nx, ny, kind_x=kx, kind_y=ky)
    q, b = _front_state(og)
    dx = 2.0 / (nx - 1 if kx else nx)
    dt = 0.25 * dx / 20.0
    T = 40 * dt
    want, rec = orc.solve(og, Phys(9.81, 500.0, 1e-12), b, q, 0.0, T, default_cfg(fixed_dt=dt))
    g, ctx = _ctx(og, b)
    ctx.set_rows_per_block(8)
    for mode in (3, 0):
        ctx.fused_stages = mode
        res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, T, H.IntegratorConfig(fixed_dt=dt))
        assert (res.accepted, res.aborted) == (rec.accepted, bool(rec.aborted))
        assert _neq(res.q.flat(), want) == 0, f"mode {mode}"


def test_tiny_bathymetry_literal_everywhere(orc):
    """b ~ 1e-300 on part of a periodic power-of-two grid (kind 2): the
    common factor is disabled by the host check, the literal association
    runs everywhere, results stay bit-identical."""
    og = omake_grid(128, 128)
    q, _ = _front_state(og)
    _, b = _front_state(og, tiny_b=True)
    assert (np.abs(b[b != 0]) < 2.0 ** -120).any()
    dt = 0.25 * (2.0 / 128) / 20.0
    want, rec = orc.solve(og, Phys(9.81, 500.0, 1e-12), b, q, 0.0, 6 * dt, default_cfg(fixed_dt=dt))
    g, ctx = _ctx(og, b)
    assert ctx.stencil_kind == 2
    res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 6 * dt, H.IntegratorConfig(fixed_dt=dt))
    assert _neq(res.q.flat(), want) == 0


@pytest.mark.parametrize("nx,kx", [(128, 0), (96, 0), (129, 1)])
def test_sources_fused_match_per_stage_and_oracle(orc, nx, kx):
    """Manufactured forcing: the fused S12 + S3 steps against the per-stage
    structure (same device sources: bit-identical stage algebra up to the
    source term's halo rows) and against the oracle (glibc sin / cos)."""
    og = omake_grid(nx, nx, kind_x=kx, kind_y=kx)
    q, b = mms_exact_field(og, 0.0)
    dx = 2.0 / (nx - 1 if kx else nx)
    dt = 0.25 * dx / 20.0
    T = 8 * dt
    want, rec = orc.solve(og, Phys(9.81, 500.0, 1e-12), b, q, 0.0, T, default_cfg(fixed_dt=dt), source_kind=1)
    g, ctx = _ctx(og, b)
    ctx.source = "manufactured"
    outs = {}
    for mode in (3, 0):
        ctx.fused_stages = mode
        res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, T, H.IntegratorConfig(fixed_dt=dt))
        assert res.accepted == rec.accepted and not res.aborted
        outs[mode] = res.q.flat().copy()
    scale = np.max(np.abs(want))
    assert np.max(np.abs(outs[3] - outs[0])) <= 1e-13 * scale
    assert np.max(np.abs(outs[3] - want)) <= 1e-12 * scale


def test_sources_adaptive_fused(orc):
    og = omake_grid(96, 96)
    q, b = mms_exact_field(og, 0.0)
    cfg = default_cfg(abs_tol=1e-8, rel_tol=1e-8)
    want, rec = orc.solve(og, Phys(9.81, 500.0, 1e-12), b, q, 0.0, 0.01, cfg, source_kind=1)
    g, ctx = _ctx(og, b)
    ctx.source = "manufactured"
    res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 0.01, H.IntegratorConfig(abs_tol=1e-8, rel_tol=1e-8))
    assert not res.aborted and abs(res.accepted - rec.accepted) <= 1
    assert np.max(np.abs(res.q.flat() - want)) <= 1e-9 * np.max(np.abs(want))
