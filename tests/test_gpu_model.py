"""GPU: the reference's test_model.cpp and test_analysis.cpp cases for the
diagnostics and init_auxiliary that run on the device (total_mass,
total_energy, energy_rate, discrete_l2_error, init_auxiliary), with the
reference test's expected values and tolerances."""
import math

import numpy as np
import pytest

import paper_2601_02540_b200 as H

pytestmark = pytest.mark.gpu

P, B = H.BoundaryKind.periodic, H.BoundaryKind.bounded


def _ctx(g, b=None, lam=500.0):
    b = np.zeros((g.ny, g.nx)) if b is None else b
    return H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b))


def test_totals_reduce_to_closed_form_integrals():
    """test_model.cpp:70-101"""
    g = H.make_grid(0.0, 1.0, 0.0, 1.0, 12, 12)
    ctx = _ctx(g)
    q = H.StateField(g)
    q.h[:] = 2.0
    q.eta[:] = q.h
    assert abs(H.total_mass(ctx, q) - 2.0) <= 1e-14
    assert abs(H.total_energy(ctx, q) - 19.62) <= 1e-12  # (g/2) h^2
    g2 = H.make_grid(-1.0, 1.0, -1.0, 1.0, 9, 9, B, B)
    q2 = H.StateField(g2)
    q2.h[:] = 2.0
    assert abs(H.total_mass(_ctx(g2), q2) - 8.0) <= 1e-13
    g3 = H.make_grid(0.0, 1.0, 0.0, 1.0, 32, 4)
    q3 = H.StateField(g3)
    q3.h[:] = g3.sample(lambda x, y: 1.0 + np.sin(2.0 * np.pi * x))
    assert abs(H.total_mass(_ctx(g3), q3) - 1.0) <= 1e-14


def test_auxiliary_initialization_sits_on_the_equilibrium_manifold():
    """test_model.cpp:103-145"""
    g = H.make_grid(0.0, 1.0, 0.0, 1.0, 9, 9, B, B)
    ctx = _ctx(g)
    q = H.StateField(g)
    q.h[:] = g.sample(lambda x, y: 1.0 + 0.1 * x * y)
    H.init_auxiliary(ctx, q)
    assert np.array_equal(q.eta, q.h) and np.all(q.w == 0.0)
    q = H.StateField(g)
    q.h[:], q.u[:], q.v[:] = 1.5, 0.7, -0.3
    H.init_auxiliary(ctx, q)
    assert np.all(q.w == 0.0)
    q = H.StateField(g)
    q.h[:] = 2.0
    q.u[:] = g.sample(lambda x, y: x + 0 * y)
    H.init_auxiliary(ctx, q)
    assert np.all(np.abs(q.w + 2.0) <= 1e-12)
    slope = g.sample(lambda x, y: 0.2 * x + 0 * y)
    ctx2 = _ctx(g, slope)
    q = H.StateField(g)
    q.h[:], q.u[:] = 1.0, 0.4
    H.init_auxiliary(ctx2, q)
    assert np.all(np.abs(q.w - 1.5 * 0.4 * 0.2) <= 1e-13)


def test_weighted_error_norm_of_elementary_differences():
    """test_analysis.cpp:27-56"""
    g = H.make_grid(0.0, 1.0, 0.0, 1.0, 5, 5, B, B)
    ctx = _ctx(g)

    def l2(a, b):  # field 0 of two states
        qa, qb = H.StateField(g), H.StateField(g)
        qa.h[:], qb.h[:] = a, b
        return H.discrete_l2_error(ctx, qa, qb, 0)
    a = g.sample(lambda x, y: np.sin(x) * y)
    assert l2(a, a) == 0.0
    c, z = np.full((5, 5), 3.25), np.zeros((5, 5))
    assert abs(l2(c, z) - 3.25) <= 1e-14 * 3.25 and abs(l2(z, c) - 3.25) <= 1e-14 * 3.25
    ramp = g.sample(lambda x, y: x + 0 * y)
    got = l2(ramp, z)
    assert abs(got - math.sqrt(0.34375)) <= 1e-14 * got and abs(got - math.sqrt(1.0 / 3.0)) <= 0.01
    fa = g.sample(lambda x, y: x * x - y)
    fb = g.sample(lambda x, y: np.cos(3 * x + y))
    fc = g.sample(lambda x, y: x + 2 * y * y)
    assert l2(fa, fc) <= l2(fa, fb) + l2(fb, fc) + 1e-14


def test_energy_rate_is_the_directional_derivative_of_the_total_energy():
    """test_analysis.cpp:72-120: zero direction -> 0; doubling the direction
    doubles the rate exactly; central differences of the energy agree."""
    g = H.make_grid(-1.0, 1.0, -1.0, 1.0, 10, 9, B, P)
    ctx = _ctx(g, g.sample(lambda x, y: 0.05 * np.cos(x + y)))
    q, qt = H.StateField(g), H.StateField(g)
    q.h[:] = g.sample(lambda x, y: 1.0 + 0.2 * np.sin(2 * x - y))
    q.u[:] = g.sample(lambda x, y: 0.3 * np.cos(x) + 0 * y)
    q.v[:] = g.sample(lambda x, y: 0.2 * np.sin(y) + 0 * x)
    q.w[:] = g.sample(lambda x, y: 0.1 * x * y)
    q.eta[:] = g.sample(lambda x, y: 1.0 + 0.1 * np.cos(x * y))
    qt.h[:] = g.sample(lambda x, y: np.cos(x) * np.sin(y))
    qt.u[:] = g.sample(lambda x, y: np.sin(3 * x) + 0 * y)
    qt.v[:] = g.sample(lambda x, y: y + 0 * x)
    qt.w[:] = g.sample(lambda x, y: 1.0 - x + 0 * y)
    qt.eta[:] = g.sample(lambda x, y: x + y)
    assert H.energy_rate(ctx, q, H.StateField(g)) == 0.0
    r1 = H.energy_rate(ctx, q, qt)
    assert H.energy_rate(ctx, q, H.StateField(g, 2.0 * qt.flat())) == 2.0 * r1
    eps = 1e-7
    ep = H.total_energy(ctx, H.StateField(g, q.flat() + eps * qt.flat()))
    em = H.total_energy(ctx, H.StateField(g, q.flat() - eps * qt.flat()))
    assert abs((ep - em) / (2 * eps) - r1) <= 1e-6 * max(1.0, abs(r1))
