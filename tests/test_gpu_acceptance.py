"""GPU: the reference acceptance gates that exercise the physics of the path
(acceptance_main.cpp c5-c9), run on the device with initial states from the
reference's own scenario library (oracle/_ref: make_scenario + prepare_run)
or, for the convergence gates, from the product's own registry and
refinement driver (scenarios.py, cli.run_convergence_study).

c5  solitary wave {200, 400, 800} x 4, lambda = 30000, tol 1e-10: orders of
    h, u at the finest pair in (1.8, 2.2)
c6  manufactured solution {32, 64, 128}^2, periodic and reflecting, tol
    1e-10: orders of all five fields at the finest pair in (1.8, 2.2)

c7  dam break: plateau depth within 0.02 and leading crest within 0.04 of
    riemann_predictions(1.8, 1.0, g) (scenarios.hpp:410-428)
c8  solitary wave against a wall: runup in [0.15, 0.195] for amplitude
    0.075; the returning crest within 0.0075 of 0.075 (gauges and the
    snapshot rule of the on-device recorder)
c9  tightening the step tolerance (1e-4 -> 1e-8) tightens the fully
    discrete energy drift (head-on soliton collision)
The per-RHS linear-cost gate (c10) is a CPU-threading property and has no
device analogue (small grids are launch-latency bound on a GPU).
"""
import math

import numpy as np
import pytest

from oracle_lib import Oracle, ref_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")]

import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200 import recorder as R  # noqa: E402


@pytest.fixture(scope="module")
def ref():
    return Oracle("ref")


def _device_run(ref, name):
    g, ph, b, q0, sk, t0, tf = ref.prepare(name)
    grid = H.make_grid(g.x_min, g.x_max, g.y_min, g.y_max, g.nx, g.ny, g.kind_x, g.kind_y)
    ctx = H.make_rhs_context(grid, H.PhysSetup(ph.g, ph.lambda_, ph.h_floor, b.reshape(g.ny, g.nx)))
    assert sk == 0
    return grid, ctx, q0, t0, tf, ph.g


def test_c7_riemann_plateau_and_crest(ref):
    grid, ctx, q0, t0, tf, g = _device_run(ref, "riemann")
    sol = H.adaptive_solve(ctx, H.StateField(grid, q0), t0, tf, H.IntegratorConfig())
    assert not sol.aborted, sol.abort_reason
    h = sol.q.h[0]  # row j = 0
    x = grid.x(np.arange(grid.nx))
    sl, sr = math.sqrt(1.8), math.sqrt(1.0)
    h_star = 0.25 * (sl + sr) ** 2
    d0 = abs(1.8 - 1.0)
    h_crest_pred = 1.0 + (d0 - d0 * d0 / 12.0)
    plateau = np.median(h[(x >= -100.0) & (x <= -20.0)])
    sel = np.flatnonzero((x >= 0.0) & (x <= 590.0))
    sel = sel[(sel >= 1) & (sel <= grid.nx - 2)]
    im = sel[np.argmax(h[sel])]
    hm, h0, hp = h[im - 1], h[im], h[im + 1]
    den = hm - 2.0 * h0 + hp
    crest = h0 - (hp - hm) ** 2 / (8.0 * den) if den < 0.0 else h0
    assert abs(plateau - h_star) <= 0.02, (plateau, h_star)
    assert abs(crest - h_crest_pred) <= 0.04, (crest, h_crest_pred)


def test_c8_wall_reflection_runup(ref, tmp_path):
    grid, ctx, q0, t0, tf, g = _device_run(ref, "wall_reflection")
    eps = 0.075
    speed = math.sqrt(g * 1.0 * (1.0 + eps))  # soliton_shape (scenarios.hpp:93-103)
    t_return = 100.0 / speed
    wall = [(grid.x_max, grid.y(j)) for j in range(grid.ny)]  # gauges on the wall column
    rec = R.RunRecorder(ctx, str(tmp_path), wall, [t_return], 1 << 40)
    sol = H.adaptive_solve(ctx, H.StateField(grid, q0), t0, tf, H.IntegratorConfig(), recorder=rec)
    assert not sol.aborted, sol.abort_reason
    nodes = rec.gauge_nodes()
    assert all(n.i == grid.nx - 1 for n in nodes)
    t, v = rec.gauge_series()  # h + b with b = 0
    runup = float(np.max(v - 1.0))
    _, actual, qs = rec.snapshot_state(0)
    back = float(np.max(qs[:grid.nx * grid.ny] - 1.0))
    assert 0.15 <= runup <= 0.195, runup
    assert abs(back - 0.075) <= 0.0075, (back, actual)


def test_c9_energy_drift_shrinks_with_tolerance(ref):
    grid, ctx, q0, t0, tf, g = _device_run(ref, "head_on_collision")
    e0 = H.total_energy(ctx, H.StateField(grid, q0))
    drift = []
    for tol in (1e-4, 1e-8):
        sol = H.adaptive_solve(ctx, H.StateField(grid, q0), t0, tf, H.IntegratorConfig(abs_tol=tol, rel_tol=tol))
        assert not sol.aborted, sol.abort_reason
        drift.append(abs(H.total_energy(ctx, sol.q) - e0) / e0)
    assert drift[1] < drift[0], drift


def test_c5_soliton_order():
    """acceptance_main.cpp:162-178 on the device."""
    from paper_2601_02540_b200 import cli
    from paper_2601_02540_b200.scenarios import make_scenario
    spec = make_scenario("soliton")
    t = cli.run_convergence_study(spec, [200, 400, 800], H.IntegratorConfig(abs_tol=1e-10, rel_tol=1e-10),
                                  ny_fixed=4)
    assert t.status == ["ok"] * 3 and t.variables == ["h", "u"]
    assert all(1.8 < r < 2.2 for r in t.rates[-1]), t.rates


@pytest.mark.parametrize("bounded", [0.0, 1.0])
def test_c6_manufactured_order(bounded):
    """acceptance_main.cpp:180-203 on the device (device forcing terms)."""
    from paper_2601_02540_b200 import cli
    from paper_2601_02540_b200.scenarios import make_scenario
    spec = make_scenario("manufactured", {"bounded": bounded})
    t = cli.run_convergence_study(spec, [32, 64, 128], H.IntegratorConfig(abs_tol=1e-10, rel_tol=1e-10))
    assert t.status == ["ok"] * 3
    assert all(1.8 < r < 2.2 for r in t.rates[-1]), t.rates
