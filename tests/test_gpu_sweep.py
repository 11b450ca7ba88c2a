"""GPU: seeded random sweep of grid shapes, boundary kinds, row-block sizes
and fixed-step kernel structures against the oracle (bitwise), plus the
in-process slab group on the same shapes.  Catches tile / row-strip / wrap /
clamp seams that the hand-picked cases in test_gpu_fused.py might miss."""
import numpy as np
import pytest

from oracle_lib import Oracle, Phys, default_cfg, make_grid as omake_grid, mms_exact_field

pytestmark = pytest.mark.gpu

import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200.slab import SlabGroup  # noqa: E402

_rng = np.random.default_rng(20261018)
CASES = [(int(_rng.integers(4, 300)), int(_rng.integers(4, 160)), int(_rng.integers(0, 2)), int(_rng.integers(0, 2)),
          int(_rng.choice([0, 1, 2, 3, 5, 8, 13])), int(_rng.choice([0, 3]))) for _ in range(24)]


@pytest.fixture(scope="module")
def orc():
    o = Oracle("orc")
    o.set_threads(8)
    return o


@pytest.mark.parametrize("nx,ny,kx,ky,rpb,mode", CASES)
def test_random_shapes_bitwise(orc, nx, ny, kx, ky, rpb, mode):
    og = omake_grid(nx, ny, kind_x=kx, kind_y=ky)
    q, b = mms_exact_field(og, 0.3)
    dx = 2.0 / (nx - 1 if kx else nx)
    dy = 2.0 / (ny - 1 if ky else ny)
    dt = 0.2 * min(dx, dy) / 20.0
    steps = 4
    want, rec = orc.solve(og, Phys(9.81, 500.0, 1e-12), b, q, 0.0, steps * dt, default_cfg(fixed_dt=dt))
    g = H.make_grid(-1.0, 1.0, -1.0, 1.0, nx, ny, kx, ky)
    phys = H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(ny, nx))
    ctx = H.make_rhs_context(g, phys)
    if rpb:
        ctx.set_rows_per_block(rpb)
    ctx.fused_stages = mode
    res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, steps * dt, H.IntegratorConfig(fixed_dt=dt))
    assert res.accepted == rec.accepted
    got = res.q.flat()
    assert np.count_nonzero(got != want) == 0
    # the same shape cut into slabs (two-row-thick slabs where possible)
    n = max(1, min(5, ny // 2))
    if n >= 2:
        grp = SlabGroup(g, phys, n)
        y = grp.state(q)
        k1 = grp.state()
        grp.rhs(0.0, y, k1)
        assert grp.bs3_fixed_steps(y, k1, 0.0, dt, steps) == steps
        # (the group integrates plain fixed steps; compare with the context's)
        ctx.fused_stages = 3
        yc = ctx.state(H.StateField(g, q))
        kc = ctx.state()
        H.rhs(ctx, 0.0, yc, kc)
        H.bs3_fixed_steps(ctx, yc, kc, 0.0, dt, steps)
        assert np.count_nonzero(grp.download(y) != yc.download().flat()) == 0
        grp.close()
