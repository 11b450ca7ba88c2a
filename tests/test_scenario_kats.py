"""CPU: the closed-form checks of the reference's test_scenarios.cpp on the
product's scenario registry (hsgn_scenarios.cpp through scenarios.py):
profile parameters, geometry, timing tables, jump conditions, registry
overrides.  The same tolerances as the reference test (Catch::Approx
epsilon / margin)."""
import math

import numpy as np
import pytest

from paper_2601_02540_b200 import scenarios as S


def approx(a, b, eps=1e-14, margin=0.0):
    return abs(a - b) <= max(margin, eps * max(abs(a), abs(b)))


def b_(spec, x, y=0.0):
    return S.evaluate(spec, x, y)[0]


def h_(spec, x, y=0.0):
    return S.evaluate(spec, x, y)[1]


def u_(spec, x, y=0.0):
    return S.evaluate(spec, x, y)[2]


def test_travelling_solitary_wave():
    """test_scenarios.cpp:58-90"""
    spec = S.make_scenario("soliton")
    eps = 0.2
    speed = math.sqrt(9.81 * 1.0 * (1.0 + eps))
    assert spec.lambda_ == 30000.0 and spec.exact_vars == ["h", "u"]
    assert approx(spec.t_final * speed, 60.0)
    g = spec.grid(32, 4)
    a, b = S.exact_state(spec, 32, 4, 0.0), S.exact_state(spec, 32, 4, spec.t_final)
    n = 32 * 4
    assert np.allclose(b[:n], a[:n], rtol=1e-12, atol=0)
    sy = S.make_scenario("soliton", {"axis": 1})
    assert sy.exact_vars == ["h", "v"] and sy.nx_default == 4
    _, q = S.sample_initial(sy, 4, 64)
    assert np.all(q[4 * 64:2 * 4 * 64] == 0.0)  # u is zero for the transverse variant
    assert g.nx == 32


def test_submerged_bar_geometry():
    """test_scenarios.cpp:164-202"""
    spec = S.make_scenario("dingemans")
    assert b_(spec, 0.0) == 0.0 and b_(spec, 11.01) == 0.0 and b_(spec, 25.0) == 0.6 and b_(spec, 35.0) == 0.0
    assert approx(b_(spec, 30.0), 0.6 * 3.07 / 6.03)
    for xb in (11.01, 23.04, 27.04, 33.07):
        assert abs(b_(spec, xb - 1e-9) - b_(spec, xb + 1e-9)) <= 1e-8
    assert approx(h_(spec, 25.0), 0.2) and u_(spec, 25.0) == 0.0
    omega = 2.0 * math.pi / 2.02
    k = omega / math.sqrt(9.81 * 0.8)
    for _ in range(100):  # dispersion_wavenumber (scenarios.hpp:223-238)
        th = math.tanh(k * 0.8)
        step = (9.81 * k * th - omega * omega) / (9.81 * th + 9.81 * k * 0.8 * (1 - th * th))
        k -= step
        if abs(step) <= 1e-15 * k:
            break
    c = omega / k
    for x in (-50.0, -30.0, -72.5):
        zeta = h_(spec, x, -46.0) - 0.8 + b_(spec, x, -46.0)
        assert abs(zeta) <= 0.02 + 1e-12
        assert approx(u_(spec, x, -46.0), c * zeta / 0.8, eps=0, margin=1e-12)
    assert len(spec.gauges) == 6 and spec.gauges[0][0] == 3.04 and spec.gauges[-1][0] == 37.04
    assert all(gp[1] == -46.0 for gp in spec.gauges)
    assert spec.nx_default == 3680 and spec.t_final == 60.0


def test_counter_propagating_solitary_waves():
    """test_scenarios.cpp:204-214"""
    spec = S.make_scenario("head_on_collision")
    assert spec.t0 == 18.5 and spec.t_final == 21.5
    assert u_(spec, 0.4) > 0.0 and u_(spec, 1.195) < 0.0
    assert h_(spec, 0.4) > 0.05 + 0.01
    assert approx(h_(spec, -10.0), 0.05, eps=0, margin=1e-10) and approx(h_(spec, 10.0), 0.05, eps=0, margin=1e-10)


def test_wall_run_timing_and_measurement_points():
    """test_scenarios.cpp:216-237"""
    spec = S.make_scenario("wall_reflection")
    assert int(spec.kind_x) == 1 and int(spec.kind_y) == 0 and spec.x_max == 0.0
    scale = math.sqrt(1.0 / 9.81)
    assert len(spec.snapshot_times) == 5
    assert approx(spec.snapshot_times[0], 24.0 * scale) and approx(spec.snapshot_times[4], 90.0 * scale)
    assert spec.gauges == [(0.0, 0.0)]
    steep = S.make_scenario("wall_reflection", {"amplitude": 0.65})
    assert steep.snapshot_times[0] == 0.0 and approx(steep.snapshot_times[4], 70.0 * scale)
    assert approx(h_(spec, -50.0), 1.075) and approx(h_(spec, -99.0), 1.0, eps=0, margin=1e-6)


def test_submerged_bump_in_two_dimensions():
    """test_scenarios.cpp:239-266"""
    spec = S.make_scenario("gaussian_obstacle")
    assert b_(spec, 0.0, 0.0) == 0.1 and approx(b_(spec, 1.0, 1.0), 0.1 * math.exp(-1.0))
    assert (spec.nx_default, spec.ny_default) == (200, 100)
    assert approx(h_(spec, 30.0, 8.0) + b_(spec, 30.0, 8.0), 0.2, eps=0, margin=1e-8)
    assert approx(h_(spec, -3.0, 5.0) + b_(spec, -3.0, 5.0), 0.2365)
    walled = S.make_scenario("gaussian_obstacle", {"bounded": 1})
    assert (walled.nx_default, walled.ny_default) == (201, 101)
    for sp in (spec, walled):
        g = sp.grid(sp.nx_default, sp.ny_default)
        assert approx(g.dx, 0.2) and approx(g.dy, 0.2)


def test_dam_break_initial_data():
    """test_scenarios.cpp:268-285 (the initial data; the shallow-water
    predictions are the acceptance gate's, tests/test_gpu_acceptance.py)"""
    spec = S.make_scenario("riemann")
    assert approx(h_(spec, 0.0), 1.4)
    assert approx(h_(spec, -600.0), 1.8, eps=0, margin=1e-12) and approx(h_(spec, 600.0), 1.0, eps=0, margin=1e-12)
    assert int(spec.kind_x) == 1


def test_smoothed_bore_front_obeys_the_jump_conditions():
    """test_scenarios.cpp:294-305"""
    eps, h0, g = 0.1, 1.0, 9.81
    spec = S.make_scenario("favre", {"eps": eps, "h0": h0})
    assert approx(h_(spec, 0.0), h0 + 0.5 * eps * h0)
    dh = h_(spec, -150.0) - h_(spec, 150.0)
    du = u_(spec, -150.0) - u_(spec, 150.0)
    assert approx(dh, eps * h0, eps=0, margin=1e-12)
    h1 = h0 + eps * h0
    assert approx(du * du * 2.0 * h0 * h1, g * (h1 + h0) * dh * dh, eps=1e-10)
    assert approx(u_(spec, 150.0), 0.0, eps=0, margin=1e-12)


@pytest.mark.parametrize("name,nx,ny", [("soliton", 64, 4), ("manufactured", 16, 16), ("dingemans", 128, 4),
                                        ("head_on_collision", 64, 4), ("wall_reflection", 64, 4),
                                        ("gaussian_obstacle", 64, 16), ("riemann", 64, 4), ("favre", 64, 4),
                                        ("still_water", 8, 8), ("lake_at_rest", 16, 16)])
def test_every_catalogued_scenario_starts_consistent(name, nx, ny):
    """test_scenarios.cpp:307-321: positive depth, finite data everywhere."""
    b, q = S.sample_initial(S.make_scenario(name), nx, ny)
    n = nx * ny
    assert np.all(np.isfinite(q)) and np.all(np.isfinite(b))
    assert np.all(q[:n] > 0.0)


def test_registry_applies_overrides_and_rejects_typos():
    """test_scenarios.cpp:323-335"""
    assert approx(h_(S.make_scenario("soliton", {"amplitude": 0.1}), 0.0), 1.1)
    assert int(S.make_scenario("manufactured", {"bounded": 1.0}).kind_x) == 1
    assert S.make_scenario("lake_at_rest", {"lambda": 42.0}).lambda_ == 42.0
    with pytest.raises(ValueError):
        S.make_scenario("no_such_flow")
    with pytest.raises(ValueError):
        S.make_scenario("soliton", {"amplitdue": 0.1})
    for name in S.scenario_names():
        S.make_scenario(name)
