"""GPU test of the multi-slab kernel path (ghost rows, slab edge modes,
per-stage halo exchange) on ONE B200: n slab contexts in one process
(hsgn_group_*), halos pulled by an event-ordered copy kernel -- the same
schedule the NCCL path runs across GPUs.  Required: bitwise equality with the
single-context run (the RHS has no reductions), and decomposition-independent
SBP-norm diagnostics (row sums combined in global row order)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200 import slab as S  # noqa: E402
from paper_2601_02540_b200.workloads import mms_fields  # noqa: E402


@pytest.mark.parametrize("n,kind_y,ny", [(2, 0, 70), (3, 0, 70), (4, 1, 70), (3, 1, 70), (5, 0, 70),
                                         (5, 0, 10), (5, 1, 10), (4, 0, 9)])
def test_group_matches_single_context_bitwise(n, kind_y, ny):
    """(ny = 10, 9 with 4-5 slabs: slabs of 2-3 rows, i.e. as thin as the two
    ghost rows the fused S12 kernel reads across a slab edge.)"""
    nx = 96
    g, q, b = mms_fields(nx, ny, 0.3, kind_y=H.BoundaryKind(kind_y))
    phys = H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(ny, nx))
    ctx = H.make_rhs_context(g, phys)
    dt = 0.25 * g.dx / 20.0
    # single context reference
    y1 = ctx.state(q)
    k1 = ctx.state()
    H.rhs(ctx, 0.0, y1, k1)
    k1_host = k1.download().flat().copy()
    H.bs3_fixed_steps(ctx, y1, k1, 0.0, dt, 9)
    want_y, want_k = y1.download().flat(), k1.download().flat()
    # n slabs on the same GPU
    grp = S.SlabGroup(g, phys, n)
    gy, gk = grp.state(q), grp.state()
    grp.rhs(0.0, gy, gk)
    assert np.count_nonzero(grp.download(gk) != k1_host) == 0
    assert grp.bs3_fixed_steps(gy, gk, 0.0, dt, 9) == 9
    assert np.count_nonzero(grp.download(gy) != want_y) == 0
    assert np.count_nonzero(grp.download(gk) != want_k) == 0
    # decomposition-independent diagnostics
    qs = H.StateField(g, want_y)
    assert grp.reduce(0, gy) == H.total_mass(ctx, qs)
    assert grp.reduce(1, gy) == H.total_energy(ctx, qs)
    assert grp.reduce(2, gy, gk) == H.energy_rate(ctx, qs, H.StateField(g, want_k))
    grp.close()


def test_group_with_manufactured_source_and_walls():
    """global row index of every slab (source terms) and wall closures on
    the first/last slab only."""
    nx, ny = 64, 48
    g, q, b = mms_fields(nx, ny, 0.3, kind_x=H.BoundaryKind.bounded, kind_y=H.BoundaryKind.bounded)
    phys = H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(ny, nx))
    ctx = H.make_rhs_context(g, phys)
    out = H.StateField(g)
    H.rhs(ctx, 0.0, H.StateField(g, q), out)
    grp = S.SlabGroup(g, phys, 3)
    gy, go = grp.state(q), grp.state()
    grp.rhs(0.0, gy, go)
    assert np.count_nonzero(grp.download(go) != out.flat()) == 0
    grp.close()


def test_group_halts_when_one_slab_goes_dry():
    """A depth failure that only one slab sees (a draining hole inside slab
    0 of 3) halts every slab at the same step: the steps done and the last
    valid state equal the single-context run's (a failure local
    to one slab must not let the other slabs step on)."""
    nx, ny, n = 64, 48, 3
    x = -1 + np.arange(nx) * 2 / nx
    y = -1 + np.arange(ny) * 2 / ny
    X, Y = np.meshgrid(x, y)
    e = np.exp(-(X ** 2 + (Y + 0.7) ** 2) / 0.02)
    h = 1 - 0.99 * e
    q = np.concatenate([h.ravel(), (10 * X * e).ravel(), (10 * (Y + 0.7) * e).ravel(), np.zeros(nx * ny),
                        h.ravel()])
    g = H.make_grid(-1.0, 1.0, -1.0, 1.0, nx, ny)
    phys = H.PhysSetup(9.81, 500.0, 1e-12, np.zeros((ny, nx)))
    dt, steps = 1e-3, 200
    ctx = H.make_rhs_context(g, phys)
    a = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, steps * dt, H.IntegratorConfig(fixed_dt=dt))
    assert a.aborted and 0 < a.accepted < steps

    N = H.api.N
    grp = S.SlabGroup(g, phys, n)
    gy, gk = grp.state(q), grp.state()
    grp.rhs(0.0, gy, gk)
    done = C.c_int64(0)
    st = N.lib().hsgn_group_bs3_fixed_steps(grp._h, gy, gk, 0.0, dt, steps, C.byref(done))
    assert st == N.HSGN_EDEPTH
    assert done.value == a.accepted
    assert np.count_nonzero(grp.download(gy) != a.q.flat()) == 0
    grp.close()
    ctx.close()
