"""Run recorder: the on-device RunRecorder against the
reference's own RunRecorder (io.hpp:107-219, driven as in cli.hpp:100-116 by
oracle/_ref's ref_run_recorded), compared through the CSV files both write.

Fixed-step runs are the bitwise path: gauges.csv and every snapshot CSV must
be byte-identical to the reference's; conservation.csv has identical times
and row count, and values within the reductions' tolerance (the device sums
rows in double-double, the reference with two-level Kahan: DESIGN.md 3).
"""
import os

import numpy as np
import pytest

from oracle_lib import Oracle, Phys, default_cfg, make_grid as omake_grid, mms_exact_field, ref_available

import paper_2601_02540_b200 as H
from paper_2601_02540_b200 import recorder as R

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")

GAUGES = [(0.1, 0.2), (-0.5, 0.77), (0.99, -1.0), (3.0, 3.0)]  # the last clamps to the corner node


def _case(nx=48, ny=40, kind=0):
    og = omake_grid(nx, ny, kind_x=kind, kind_y=kind)
    q, b = mms_exact_field(og, 0.3)
    grid = H.make_grid(-1.0, 1.0, -1.0, 1.0, nx, ny, kind, kind)
    return og, grid, q, b


def _read(path):
    with open(path) as f:
        return f.read()


def _cons(path):
    a = np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)
    return a


# ------------------------------------------------------------------ CPU (host formatting)

@needs_ref
def test_snapshot_and_gauge_format_match_reference(tmp_path):
    """write_snapshot_csv / nearest_node / fmt17 reproduce the reference's
    files byte for byte (host-side formatting, no GPU)."""
    og, grid, q, b = _case(24, 20, kind=1)
    ref = Oracle("ref")
    ref.set_threads(4)
    ph = Phys(9.81, 500.0, 1e-12)
    cfg = default_cfg(fixed_dt=1e-3)
    _, rec = ref.run_recorded(og, ph, b, q, 0.0, 8e-3, cfg, str(tmp_path / "a"))
    # a target at the final time snapshots the final state (io.hpp:126-129)
    qf, rec2 = ref.run_recorded(og, ph, b, q, 0.0, 8e-3, cfg, str(tmp_path / "b"), gauges=GAUGES,
                                targets=[rec.t], stride=2)
    assert rec2.t == rec.t
    name = "snapshot_t" + R.fmt_short(rec.t) + ".csv"
    mine = tmp_path / "mine.csv"
    R.write_snapshot_csv(str(mine), grid, qf, b)
    assert _read(mine) == _read(tmp_path / "b" / name)
    head = [ln for ln in _read(tmp_path / "b" / "gauges.csv").splitlines() if ln.startswith("#")]
    nodes = [R.nearest_node(grid, x, y) for x, y in GAUGES]
    assert head == [f"# gauge_{k + 1} at ({R.fmt17(n.x)}, {R.fmt17(n.y)})" for k, n in enumerate(nodes)]


# ------------------------------------------------------------------ GPU

def _run_both(tmp_path, og, grid, q, b, cfg_kw, t_final, targets, stride, lam=500.0):
    ref = Oracle("ref")
    ref.set_threads(8)
    ph = Phys(9.81, lam, 1e-12)
    rdir, ddir = str(tmp_path / "ref"), str(tmp_path / "dev")
    qr, rr = ref.run_recorded(og, ph, b, q, 0.0, t_final, default_cfg(**cfg_kw), rdir, gauges=GAUGES,
                              targets=targets, stride=stride)
    ctx = H.make_rhs_context(grid, H.PhysSetup(g=9.81, lambda_=lam, b=b.reshape(grid.ny, grid.nx)))
    rec = R.RunRecorder(ctx, ddir, GAUGES, targets, stride)
    sol = H.adaptive_solve(ctx, H.StateField(grid, q), 0.0, t_final, H.IntegratorConfig(**cfg_kw), recorder=rec)
    rec.flush()
    return rdir, ddir, qr, rr, sol, rec


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("kind,stride", [(0, 3), (1, 1), (1, 8)])
def test_recorder_fixed_step_matches_reference(tmp_path, kind, stride):
    og, grid, q, b = _case(kind=kind)
    dt = 1e-3
    t_final = 37 * dt
    # before t0 (initial state), between nodes (closer-neighbour rule both
    # ways), exactly on a step, and beyond t_final (never taken)
    targets = [-1.0, 0.00449, 0.00551, 0.02, 0.5]
    rdir, ddir, qr, rr, sol, rec = _run_both(tmp_path, og, grid, q, b, dict(fixed_dt=dt), t_final, targets,
                                             stride)
    assert sol.accepted == rr.accepted and not sol.aborted
    assert np.array_equal(sol.q.flat(), qr)
    assert _read(os.path.join(ddir, "gauges.csv")) == _read(os.path.join(rdir, "gauges.csv"))
    snaps_ref = sorted(f for f in os.listdir(rdir) if f.startswith("snapshot_"))
    snaps_dev = sorted(f for f in os.listdir(ddir) if f.startswith("snapshot_"))
    assert snaps_dev == snaps_ref and len(snaps_ref) == 4
    for f in snaps_ref:
        assert _read(os.path.join(ddir, f)) == _read(os.path.join(rdir, f)), f
    cr, cd = _cons(os.path.join(rdir, "conservation.csv")), _cons(os.path.join(ddir, "conservation.csv"))
    assert cr.shape == cd.shape and cr.shape[0] == 37 // stride + 1
    assert np.array_equal(cr[:, 0], cd[:, 0])
    np.testing.assert_allclose(cd[:, 1], cr[:, 1], rtol=1e-14)
    np.testing.assert_allclose(cd[:, 2], cr[:, 2], rtol=1e-14)
    np.testing.assert_allclose(cd[:, 3], cr[:, 3], rtol=0, atol=1e-12 * cr[0, 2])
    # the recorder's in-memory rows are what flush() wrote
    rows = rec.conservation_rows()
    assert [r.t for r in rows] == list(cd[:, 0])


@pytest.mark.gpu
@needs_ref
def test_recorder_adaptive_matches_reference(tmp_path):
    og, grid, q, b = _case(kind=1)
    targets = [0.0, 0.01, 0.025]
    rdir, ddir, qr, rr, sol, rec = _run_both(tmp_path, og, grid, q, b, dict(abs_tol=1e-7, rel_tol=1e-7), 0.03,
                                             targets, 2)
    assert (sol.accepted, sol.rejected) == (rr.accepted, rr.rejected)
    gr = np.loadtxt(os.path.join(rdir, "gauges.csv"), delimiter=",", comments="#", skiprows=len(GAUGES) + 1)
    gd = np.loadtxt(os.path.join(ddir, "gauges.csv"), delimiter=",", comments="#", skiprows=len(GAUGES) + 1)
    assert gr.shape == gd.shape
    np.testing.assert_allclose(gd, gr, rtol=1e-11, atol=0)
    cr, cd = _cons(os.path.join(rdir, "conservation.csv")), _cons(os.path.join(ddir, "conservation.csv"))
    assert cr.shape == cd.shape
    np.testing.assert_allclose(cd[:, :3], cr[:, :3], rtol=1e-11)
    snaps = rec.snapshots()
    assert [s.target for s in snaps] == targets
    ref_names = sorted(f for f in os.listdir(rdir) if f.startswith("snapshot_"))
    assert sorted(os.path.basename(s.path) for s in snaps) == ref_names


@pytest.mark.gpu
def test_recorder_keeps_graph_chunks_and_counts():
    """A stride-16 recorder on a fixed-step run: rows at k*16 (k = 0, 1, ...),
    one gauge row per accepted step plus the initial one, and the device
    conservation row equals the standalone reductions of the final state."""
    _, grid, q, b = _case(64, 64)
    ctx = H.make_rhs_context(grid, H.PhysSetup(g=9.81, lambda_=500.0, b=b.reshape(64, 64)))
    rec = R.RunRecorder(ctx, "/tmp/unused", [(0.0, 0.0)], [], 16)
    sol = H.adaptive_solve(ctx, H.StateField(grid, q), 0.0, 64e-4, H.IntegratorConfig(fixed_dt=1e-4),
                           recorder=rec)
    assert sol.accepted == 64
    t, v = rec.gauge_series()
    assert len(t) == 65 and v.shape == (65, 1)
    rows = rec.conservation_rows()
    assert len(rows) == 5
    last = rows[-1]
    assert last.t == sol.t
    assert last.mass == H.total_mass(ctx, sol.q)
    assert last.energy == H.total_energy(ctx, sol.q)


@pytest.mark.gpu
def test_recorder_rejects_bad_stride():
    _, grid, q, b = _case(16, 16)
    ctx = H.make_rhs_context(grid, H.PhysSetup(g=9.81, lambda_=500.0, b=b.reshape(16, 16)))
    with pytest.raises(ValueError):
        R.RunRecorder(ctx, "/tmp/unused", [], [], 0)
