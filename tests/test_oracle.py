"""CPU tests of the oracle (oracle/hsgn_oracle.c): pinned to the reference.

1. Against the committed golden vectors (tests/golden/golden_r1.npz, made by
   oracle/make_golden.py from the unmodified reference): bit-for-bit.
2. Against the reference compiled in place (oracle/_ref), when present:
   bit-for-bit on extra randomised cases.
3. The reference's own known-answer tests for this path (SURVEY.md section
   4 table), restated: SBP stencil / mass / SAT KATs, manufactured KATs,
   well-balancedness, conservation, decoupling, failure path.
"""
import os

import numpy as np
import pytest

from oracle_lib import (Oracle, Phys, default_cfg, make_grid, mms_exact_field, random_state, ref_available,
                        same_bits)

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_r1.npz")


@pytest.fixture(scope="module")
def orc():
    o = Oracle("orc")
    o.set_threads(4)
    return o


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def grid_of(a):
    return make_grid(int(a[0]), int(a[1]), a[4], a[5], a[6], a[7], int(a[2]), int(a[3]))


def rhs_names(gold):
    return sorted({k.split("/")[1] for k in gold if k.startswith("rhs/")})


# ---------------------------------------------------------------- golden

def test_golden_rhs_bitwise(orc, gold):
    names = rhs_names(gold)
    assert len(names) >= 10
    for name in names:
        g = grid_of(gold[f"rhs/{name}/grid"])
        lam, t, source, variant = gold[f"rhs/{name}/par"]
        st, out, _ = orc.rhs(g, Phys(9.81, lam, 1e-12), gold[f"rhs/{name}/b"], gold[f"rhs/{name}/q"], t=t,
                             source_kind=int(source), variant=int(variant))
        assert st == 0
        want = gold[f"rhs/{name}/out"]
        if source:  # independently derived source closed form: ~1e-15 relative
            assert np.max(np.abs(out - want)) <= 1e-13 * np.max(np.abs(want)), name
        else:
            assert same_bits(out, want), name


def test_golden_fixed_step_bitwise(orc, gold):
    for kind in (0, 1):
        g = grid_of(gold[f"fixed/{kind}/grid"])
        dt, T = gold[f"fixed/{kind}/par"]
        q, rec = orc.solve(g, Phys(9.81, 500.0, 1e-12), gold[f"fixed/{kind}/b"], gold[f"fixed/{kind}/q0"], 0.0, T,
                           default_cfg(fixed_dt=dt))
        r = gold[f"fixed/{kind}/rec"]
        assert (rec.t, rec.accepted, rec.rejected, rec.rhs_evals) == (r[0], r[1], r[2], r[3])
        assert same_bits(q, gold[f"fixed/{kind}/q"])


def test_golden_adaptive_bitwise(orc, gold):
    g = grid_of(gold["adaptive/grid"])
    q, rec = orc.solve(g, Phys(9.81, 500.0, 1e-12), gold["adaptive/b"], gold["adaptive/q0"], 0.0, 0.01,
                       default_cfg())
    r = gold["adaptive/rec"]
    assert (rec.t, rec.accepted, rec.rejected, rec.rhs_evals, rec.rhs_evals_setup) == tuple(r[:5])
    assert same_bits(q, gold["adaptive/q"])


def test_golden_diagnostics(orc, gold):
    for name in ("periodic_random", "bounded_random", "mms_state"):
        g = grid_of(gold[f"rhs/{name}/grid"])
        lam = gold[f"rhs/{name}/par"][0]
        ph = Phys(9.81, lam, 1e-12)
        q, b, qt = gold[f"rhs/{name}/q"], gold[f"rhs/{name}/b"], gold[f"rhs/{name}/out"]
        m, e, r = gold[f"diag/{name}"]
        assert orc.total_mass(g, q) == m
        assert orc.total_energy(g, ph, b, q) == e
        assert orc.energy_rate(g, ph, b, q, qt) == r


def test_golden_init_auxiliary(orc, gold):
    for kind in (0, 1):
        g = make_grid(33, 33, -5.0, 5.0, -5.0, 5.0, kind, kind)
        b = gold[f"rhs/lake_at_rest{kind}/b"]
        q = np.zeros(5 * 33 * 33)
        q[: 33 * 33] = 1.0 - b
        assert same_bits(orc.init_auxiliary(g, b, q), gold[f"init_aux/lake{kind}/q"])


def test_golden_manufactured_kats(orc, gold):
    for p, s, sdt, src in zip(gold["mms/points"], gold["mms/state"], gold["mms/state_dt"], gold["mms/source"]):
        np.testing.assert_allclose(orc.mms_state(*p), s, rtol=1e-13, atol=1e-14)
        np.testing.assert_allclose(orc.mms_state_dt(*p), sdt, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(orc.mms_source(*p), src, rtol=1e-12, atol=1e-13)
        assert orc.mms_bathymetry(p[1], p[2]) == pytest.approx(orc.mms_state(0.0, p[1], p[2])[0] * 0 +
                                                                orc.mms_bathymetry(p[1], p[2]))


def test_manufactured_20_digit_kats(orc):
    """test_scenarios.cpp:92-136 frozen samples (tolerance 1e-13 there)."""
    tol = 1e-13
    q = orc.mms_state(0.3, 0.2, -0.4)
    assert q[0] == pytest.approx(2.1163728757031315720, rel=tol)
    assert q[1] == pytest.approx(0.27135254915624211362, rel=tol)
    assert q[2] == pytest.approx(-0.16770509831248422723, rel=tol)
    assert q[3] == pytest.approx(1.8970100851837198538, rel=tol)
    qt = orc.mms_state_dt(0.3, 0.2, -0.4)
    assert qt[0] == pytest.approx(1.6702489564306173647, rel=tol)
    assert qt[1] == pytest.approx(-0.55397454914713702718, rel=tol)
    assert qt[2] == pytest.approx(0.34237510027532975613, rel=tol)
    assert qt[3] == pytest.approx(-2.3756771873121311225, rel=tol)
    s = orc.mms_source(0.3, 0.2, -0.4, 9.81)
    assert s[0] == pytest.approx(-0.30418142560921477283, rel=tol)
    assert s[1] == pytest.approx(1.3261733514586429765, rel=tol)
    assert s[2] == pytest.approx(7.9132602466100860130, rel=tol)
    assert s[3] == pytest.approx(6.4183979930781656234, rel=tol)
    assert s[4] == pytest.approx(s[0], rel=1e-14)
    q0 = orc.mms_state(0.0, 0.3, 0.7)
    assert q0[0] == pytest.approx(1.5139260912937620925, rel=tol)
    assert q0[1] == 0.0 and q0[2] == 0.0
    s0 = orc.mms_source(0.0, 0.3, 0.7, 9.81)
    assert abs(s0[0]) <= 1e-14
    assert s0[1] == pytest.approx(10.850183177400623961, rel=tol)
    assert s0[3] == pytest.approx(10.590466100678328156, rel=tol)
    assert orc.mms_bathymetry(0.25, 0.25) == pytest.approx(0.04, rel=tol)
    assert orc.mms_state(0.0, 0.25, 0.25)[0] == pytest.approx(2.46, rel=tol)


# ------------------------------------------------------- live reference

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("nx,ny,kx,ky,lam,seed", [(31, 17, 0, 0, 500.0, 1), (16, 29, 1, 1, 30000.0, 2),
                                                   (40, 36, 1, 0, 500.0, 3), (36, 40, 0, 1, 0.0, 4),
                                                   (4, 4, 0, 0, 500.0, 5), (5, 4, 1, 1, 500.0, 6)])
def test_live_reference_rhs_bitwise(orc, nx, ny, kx, ky, lam, seed):
    ref = Oracle("ref")
    g = make_grid(nx, ny, kind_x=kx, kind_y=ky)
    q = random_state(nx * ny, seed)
    b = 0.05 * np.cos(np.arange(nx * ny) * 0.11)
    a = ref.rhs(g, Phys(9.81, lam, 1e-12), b, q)
    o = orc.rhs(g, Phys(9.81, lam, 1e-12), b, q)
    assert a[0] == o[0] == 0
    assert np.array_equal(a[1], o[1])


@needs_ref
def test_live_reference_solve_paths(orc):
    ref = Oracle("ref")
    g = make_grid(20, 16, kind_x=1, kind_y=0)
    q, b = mms_exact_field(g, 0.3)
    for cfg in [default_cfg(fixed_dt=2e-4), default_cfg(abs_tol=1e-9, rel_tol=1e-9), default_cfg(max_steps=3),
                default_cfg(dt_initial=1e-3)]:
        qa, ra = ref.solve(g, Phys(9.81, 500.0, 1e-12), b, q, 0.0, 0.005, cfg)
        qb, rb = orc.solve(g, Phys(9.81, 500.0, 1e-12), b, q, 0.0, 0.005, cfg)
        assert (ra.t, ra.accepted, ra.rejected, ra.rhs_evals, ra.aborted) == \
               (rb.t, rb.accepted, rb.rejected, rb.rhs_evals, rb.aborted)
        assert ra.reason == rb.reason
        assert np.array_equal(qa, qb)


@needs_ref
def test_live_reference_error_norm(orc):
    ref = Oracle("ref")
    g = make_grid(12, 10)
    n = 120
    ks = [random_state(n, s) for s in range(6)]
    a = ref.error_norm(1e-3, g, *ks, 1e-6, 1e-6)
    b = orc.error_norm(1e-3, g, *ks, 1e-6, 1e-6)
    assert a == b


# ------------------------------------------------- reference KATs (SBP)

def test_periodic_stencil_kat(orc):
    """test_sbp.cpp:25-35: sin(2 pi x) on 4 nodes -> (4, 0, -4, 0) exactly."""
    g = make_grid(4, 4, 0.0, 1.0, 0.0, 1.0)
    u = np.tile([0.0, 1.0, 0.0, -1.0], 4)
    d = orc.apply_d(g, 0, u).reshape(4, 4)
    assert np.array_equal(d[0], [4.0, 0.0, -4.0, 0.0])


def test_constants_and_linears(orc):
    """test_sbp.cpp:37-54, 121-141."""
    for kind in (0, 1):
        g = make_grid(17, 9, 0.0, 5.1, 0.0, 2.0, kind, kind)
        c = np.full(17 * 9, 5.5)
        assert np.all(orc.apply_d(g, 0, c) == 0.0) and np.all(orc.apply_d(g, 1, c) == 0.0)
    g = make_grid(6, 5, 0.0, 1.0, 0.0, 1.0, 1, 1)
    x = np.tile(np.arange(6) * 0.2, 5)
    y = np.repeat(np.arange(5) * 0.25, 6)
    f = 2 * x - 3 * y
    np.testing.assert_allclose(orc.apply_d(g, 0, f), 2.0, atol=1e-13)
    np.testing.assert_allclose(orc.apply_d(g, 1, f), -3.0, atol=1e-13)
    assert np.all(orc.apply_d(g, 0, y * y) == 0.0)


def test_sbp_identity(orc):
    """test_sbp.cpp:61-99 and acceptance c1 (acceptance_main.cpp:73-84)."""
    for n in (5, 6, 8):
        for kind in (0, 1):
            ok, r = orc.check_sbp(kind, n, 0.1)
            assert ok and r == 0.0
    for n in range(4, 65):
        for kind in (0, 1):
            assert orc.check_sbp(kind, n, 0.017)[0]


def test_sat_kats(orc):
    """test_sbp.cpp:190-220."""
    g = make_grid(11, 11, 0.0, 1.0, 0.0, 1.0, 1, 1)
    sat = orc.sat(g, np.full(121, 3.0), np.full(121, 2.0)).reshape(11, 11)
    assert sat[5, 5] == 0.0
    assert sat[5, 0] == pytest.approx(-60.0, abs=1e-10)
    assert sat[5, 10] == pytest.approx(60.0, abs=1e-10)
    assert sat[0, 5] == pytest.approx(-40.0, abs=1e-10)
    sat = orc.sat(g, np.full(121, 1.0), np.full(121, 2.0)).reshape(11, 11)
    assert sat[0, 0] == pytest.approx(-60.0, abs=1e-10)
    gx = make_grid(11, 8, 0.0, 1.0, 0.0, 1.0, 1, 0)
    satx = orc.sat(gx, np.ones(88), np.ones(88)).reshape(8, 11)
    assert satx[0, 3] == 0.0
    assert satx[3, 0] == pytest.approx(-20.0, abs=1e-10)


def test_quadrature(orc):
    """test_sbp.cpp:143-168."""
    g = make_grid(16, 16, 0.0, 1.0, 0.0, 1.0)
    assert orc.mass_weighted_sum(g, np.ones(256)) == pytest.approx(1.0, abs=1e-14)
    g = make_grid(9, 9, -1.0, 1.0, -1.0, 1.0, 1, 1)
    assert orc.mass_weighted_sum(g, np.full(81, 2.0)) == pytest.approx(8.0, abs=1e-13)
    g = make_grid(11, 11, 0.0, 1.0, 0.0, 1.0, 1, 1)
    assert orc.mass_weighted_sum(g, np.tile(np.arange(11) * 0.1, 11)) == pytest.approx(0.5, abs=1e-14)


# ------------------------------------------------ reference KATs (RHS)

def test_uniform_columns_steady(orc):
    """test_rhs.cpp:39-65."""
    g = make_grid(12, 10)
    n = 120
    q = np.concatenate([np.ones(n), np.full(n, 0.3), np.full(n, -0.7), np.zeros(n), np.ones(n)])
    st, out, _ = orc.rhs(g, Phys(9.81, 500.0, 1e-12), np.zeros(n), q)
    assert st == 0 and np.all(out == 0.0)
    g = make_grid(12, 10, kind_x=1, kind_y=1)
    q = np.concatenate([np.full(n, 2.0), np.zeros(3 * n), np.full(n, 2.0)])
    st, out, _ = orc.rhs(g, Phys(9.81, 500.0, 1e-12), np.zeros(n), q)
    assert np.all(out == 0.0)


def test_lake_at_rest(orc):
    """test_rhs.cpp:67-82 / acceptance c4: well-balanced to 1e-12 g."""
    for kind in (0, 1):
        g = make_grid(33, 33, -5.0, 5.0, -5.0, 5.0, kind, kind)
        xs = np.linspace(-5, 5, 33, endpoint=bool(kind)) if kind else -5 + np.arange(33) * (10 / 33)
        X, Y = np.meshgrid(xs, xs)
        b = (0.1 * np.exp(-(X * X + Y * Y))).ravel()
        q = np.zeros(5 * 1089)
        q[:1089] = 1.0 - b
        q = orc.init_auxiliary(g, b, q)
        _, out, _ = orc.rhs(g, Phys(9.81, 500.0, 1e-12), b, q)
        assert np.max(np.abs(out)) <= 1e-12 * 9.81


def test_mass_and_energy_conservation(orc):
    """test_rhs.cpp:84-127: 1^T M h_t ~ 0, <dE/dq, q_t>_M ~ 0 for random states."""
    for kx, ky, lam in [(0, 0, 500.0), (1, 1, 500.0), (1, 0, 500.0), (0, 0, 0.0)]:
        g = make_grid(20, 18, kind_x=kx, kind_y=ky)
        q = random_state(360, 21 + int(lam))
        b = 0.1 + 0.05 * np.sin(3 * np.arange(360) * 0.1)
        ph = Phys(9.81, lam, 1e-12)
        _, qt, _ = orc.rhs(g, ph, b, q)
        assert abs(orc.mass_weighted_sum(g, qt[:360])) <= 1e-12
        assert abs(orc.energy_rate(g, ph, b, q, qt)) <= 1e-11 * abs(orc.total_energy(g, ph, b, q))


def test_lambda_zero_decoupling_and_depth_error(orc):
    """test_rhs.cpp:129-157, 176-186."""
    g = make_grid(16, 16)
    n = 256
    q = random_state(n, 31)
    _, a, _ = orc.rhs(g, Phys(9.81, 0.0, 1e-12), np.zeros(n), q)
    q2 = q.copy()
    q2[3 * n:4 * n] += 0.37
    q2[4 * n:] *= 1.21
    _, b2, _ = orc.rhs(g, Phys(9.81, 0.0, 1e-12), np.zeros(n), q2)
    assert np.array_equal(a[:3 * n], b2[:3 * n])
    g = make_grid(8, 8)
    q = np.concatenate([np.ones(64), np.zeros(192), np.ones(64)])
    q[4 * 8 + 3] = -0.25
    st, out, _ = orc.rhs(g, Phys(9.81, 500.0, 1e-12), np.zeros(64), q, out=np.full(320, 7.0))
    assert st == 1 and np.all(out == 7.0)


def test_mms_residual_second_order(orc):
    """test_rhs.cpp:204-249: discrete residual ratio 32^2 -> 64^2 in (3.4, 4.6)."""
    def resid(n):
        g = make_grid(n, n)
        q, b = mms_exact_field(g, 0.3)
        _, out, _ = orc.rhs(g, Phys(9.81, 500.0, 1e-12), b, q, t=0.3, source_kind=1)
        dx = 2.0 / n
        x = -1 + np.arange(n) * dx
        X, Y = np.meshgrid(x, x)
        want = np.array([orc.mms_state_dt(0.3, xx, yy) for xx, yy in zip(X.ravel(), Y.ravel())]).T.ravel()
        return max(orc.discrete_l2_error(g, out[k * n * n:(k + 1) * n * n], want[k * n * n:(k + 1) * n * n])
                   for k in range(5))
    r = resid(32) / resid(64)
    assert 3.4 < r < 4.6


def test_fixed_step_third_order_and_failure_modes(orc):
    """Integrator semantics (time_integration.hpp:262-344) on the SGN RHS."""
    g = make_grid(16, 16)
    q, b = mms_exact_field(g, 0.3)
    ph = Phys(9.81, 500.0, 1e-12)
    _, rec = orc.solve(g, ph, b, q, 0.0, 0.01, default_cfg(fixed_dt=0.004))
    assert rec.accepted == 3 and rec.t == 0.01 and rec.rhs_evals == 10
    _, rec = orc.solve(g, ph, b, q, 2.0, 1.0, default_cfg())
    assert rec.aborted and b"precedes" in rec.reason
    _, rec = orc.solve(g, ph, b, q, 0.0, 1.0, default_cfg(max_steps=1, dt_initial=1e-3))
    assert rec.aborted and b"step budget exhausted" in rec.reason and rec.accepted == 1
    bad = q.copy()
    bad[5] = -1.0
    _, rec = orc.solve(g, ph, b, bad, 0.0, 1.0, default_cfg())
    assert rec.aborted and rec.reason.startswith(b"initial tendency")


def test_plain_stage_sequence_equals_fixed_solve(orc):
    """orc_bs3_fixed_steps (used by the slab and benchmark checks) is the
    adaptive_solve(fixed_dt) stage sequence: with dt = 2^-12 the time
    accumulates exactly, no step is clipped, and both agree bit for bit."""
    import ctypes as C
    from oracle_lib import PD
    g = make_grid(24, 20)
    q0, b = mms_exact_field(g, 0.3)
    dt = 2.0 ** -12
    want, rec = orc.solve(g, Phys(9.81, 500.0, 1e-12), b, q0, 0.0, 7 * dt, default_cfg(fixed_dt=dt))
    assert rec.accepted == 7
    y = q0.copy()
    k1 = np.zeros_like(q0)
    assert orc._fixed(C.byref(g), C.byref(Phys(9.81, 500.0, 1e-12)), b.ctypes.data_as(PD), y.ctypes.data_as(PD),
                      k1.ctypes.data_as(PD), 0.0, dt, 7, 1) == 0
    assert np.array_equal(y, want)
