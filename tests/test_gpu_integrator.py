"""GPU: the integrator cases of the reference's test_time_integration.cpp that
carry over to the device's own split-form RHS (the fused integrator does not
take the reference's generic callable, so the scalar decay / drain /
poisoned tendencies become states of the SGN system with the same effect),
compared against the oracle (the C restatement of time_integration.hpp)
where the reference test compares against a closed form.
"""
import numpy as np
import pytest

from oracle_lib import Oracle, Phys, default_cfg, make_grid as omake_grid

import paper_2601_02540_b200 as H
from paper_2601_02540_b200.workloads import mms_fields

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    o = Oracle("orc")
    o.set_threads(8)
    return o


def _still(n=32, depth=1.0):
    g = H.make_grid(-5.0, 5.0, -5.0, 5.0, n, n)
    q = np.zeros((5, n, n))
    q[0] = depth
    q[4] = depth
    return g, q.reshape(-1)


def test_zero_tendency_keeps_the_state_bit_for_bit():
    """test_time_integration.cpp:33-51: still water has an exactly zero
    tendency, so fixed and adaptive runs return the initial state bit for
    bit (and the adaptive run takes the growth-capped steps)."""
    g, q = _still()
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, np.zeros((32, 32))))
    fixed = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 0.5, H.IntegratorConfig(fixed_dt=0.01))
    assert not fixed.aborted and fixed.accepted == 50
    assert np.array_equal(fixed.q.flat(), q)
    ada = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 10.0, H.IntegratorConfig())
    assert not ada.aborted and ada.t == 10.0 and ada.rejected == 0
    assert np.array_equal(ada.q.flat(), q)


def test_explicit_initial_step_skips_the_startup_probe(orc):
    """test_time_integration.cpp:88-97: dt_initial > 0 means no probe RHS;
    without it, one probe evaluation (rhs_evals_setup == 1), as the oracle."""
    g, q, b = mms_fields(32, 32, 0.3)
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(32, 32)))
    a = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 1e-3, H.IntegratorConfig(dt_initial=1e-4))
    assert a.rhs_evals_setup == 0 and a.rhs_evals == 3 * (a.accepted + a.rejected) + 1
    b2 = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 1e-3, H.IntegratorConfig())
    _, rec = orc.solve(omake_grid(32, 32), Phys(9.81, 500.0, 1e-12), b, q, 0.0, 1e-3, default_cfg())
    assert b2.rhs_evals_setup == rec.rhs_evals_setup == 1
    assert (b2.accepted, b2.rejected) == (rec.accepted, rec.rejected)


def test_startup_estimate_shrinks_for_stiffer_tendencies():
    """test_time_integration.cpp:99-125: a stiffer tendency (larger lambda,
    faster relaxation) gives a smaller first step (the first accepted step
    time, seen by the observer)."""
    g, q, b = mms_fields(32, 32, 0.3)
    first = {}
    for lam in (50.0, 5000.0):
        ctx = H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(32, 32)))
        ts = []
        H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 1.0, H.IntegratorConfig(max_steps=1),
                         on_accept=lambda t, qd, qtd: ts.append(t))
        first[lam] = ts[1]
    assert first[5000.0] < first[50.0]


def test_degenerate_spans_terminate_immediately():
    """test_time_integration.cpp:152-163"""
    g, q = _still(8)
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, np.zeros((8, 8))))
    same = H.adaptive_solve(ctx, H.StateField(g, q), 2.0, 2.0, H.IntegratorConfig())
    assert not same.aborted and same.accepted == 0 and same.t == 2.0
    back = H.adaptive_solve(ctx, H.StateField(g, q), 2.0, 1.0, H.IntegratorConfig())
    assert back.aborted and "precedes" in back.abort_reason


@pytest.mark.parametrize("fixed", [False, True])
def test_drying_state_aborts_like_the_reference(orc, fixed):
    """test_time_integration.cpp:165-199 (drained column / stage failures):
    a nearly dry depression with converging momentum.  The adaptive run
    (floor above the initial minimum depth, the drained column) aborts on the
    depth floor; the fixed-step run aborts on a non-positive stage depth --
    with the oracle's reason, counters, time and last valid state."""
    n = 32
    x = -1 + np.arange(n) * 2 / n
    X, Y = np.meshgrid(x, x)
    e = np.exp(-(X ** 2 + Y ** 2) / 0.05)
    h = 1 - 0.999 * e
    q = np.concatenate([h.ravel(), (-40 * X * e).ravel(), (-40 * Y * e).ravel(), np.zeros(n * n), h.ravel()])
    b = np.zeros(n * n)
    # adaptive: the depression starts below the floor (drained column); fixed:
    # the converging momentum drives a stage depth negative
    kw = dict(fixed_dt=1e-3, h_floor=1e-3) if fixed else dict(dt_initial=1e-3, h_floor=0.01)
    want, rec = orc.solve(omake_grid(n, n), Phys(9.81, 500.0, 1e-12), b, q, 0.0, 0.5, default_cfg(**kw))
    assert rec.aborted
    g = H.make_grid(-1.0, 1.0, -1.0, 1.0, n, n)
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, np.zeros((n, n))))
    res = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 0.5, H.IntegratorConfig(**kw))
    assert res.aborted and res.abort_reason == rec.reason.decode()
    assert (res.accepted, res.rejected, res.rhs_evals) == (rec.accepted, rec.rejected, rec.rhs_evals)
    assert res.t == rec.t
    if fixed:
        assert np.count_nonzero(res.q.flat() != want) == 0
    else:
        assert np.allclose(res.q.flat(), want, rtol=1e-9, atol=1e-12)


def test_step_budget_reports_a_partial_result():
    """test_time_integration.cpp:201-213"""
    g, q, b = mms_fields(16, 16, 0.3)
    ctx = H.make_rhs_context(g, H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(16, 16)))
    rec = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, 100.0, H.IntegratorConfig(max_steps=1, dt_initial=1e-3))
    assert rec.aborted and "step budget exhausted" in rec.abort_reason
    assert rec.accepted == 1 and 0.0 < rec.t < 100.0
