"""CLI front end on the device (reference cli.hpp).

`hsgn run` / `converge` / `bench` (paper_2601_02540_b200.cli) against the
reference driven the same way through oracle/_ref (make_scenario +
prepare_run, adaptive_solve + RunRecorder, the convergence loop of
scenarios.hpp:535-592):
* prepare_run: the device q0 (with init_auxiliary) is bit-identical;
* fixed-step `run`: gauges.csv, every snapshot CSV and cross_section.csv
  byte-identical, conservation.csv to the reductions' tolerance, the same
  step counts and final time in run_meta.json;
* adaptive `run`: same accepted / rejected counts, values to tolerance;
* `converge`: per-rung errors equal the reference's to 1e-7 relative and the
  manufactured solution converges at second order;
* `bench` / configuration errors: files, exit codes.
"""
import json
import os

import numpy as np
import pytest

from oracle_lib import Oracle, default_cfg, ref_available

import paper_2601_02540_b200 as H
from paper_2601_02540_b200 import cli
from paper_2601_02540_b200 import recorder as R
from paper_2601_02540_b200 import scenarios as S

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


def _read(path):
    with open(path) as f:
        return f.read()


def _table(path):
    """Numeric rows of a CSV (comment lines and the header dropped)."""
    rows = [ln for ln in _read(path).splitlines() if ln and not ln.startswith("#")][1:]
    return np.array([[float(x) for x in ln.split(",")] for ln in rows]).reshape(len(rows), -1)


def _write_cfg(tmp_path, text):
    p = tmp_path / "case.cfg"
    p.write_text(text)
    return str(p)


@pytest.mark.parametrize("name,params,nx,ny", [("soliton", {"amplitude": 0.2}, 256, 4),
                                                ("gaussian_obstacle", {"bounded": 1}, 61, 31),
                                                ("manufactured", {}, 40, 36), ("lake_at_rest", {"bounded": 1}, 33, 30),
                                                ("dingemans", {}, 3680, 4)])
def test_prepare_run_bitwise(name, params, nx, ny):
    orc = Oracle("ref")
    g, ph, b, q0, *_ = orc.prepare(name, nx, ny, **params)
    run = S.prepare_run(S.make_scenario(name, params), nx, ny, device=0)
    assert np.array_equal(run.b, b)
    assert np.count_nonzero(run.q0.download().flat() != q0) == 0
    run.ctx.close()


RUN_CASES = [
    # soliton (quickstart.cfg shape) with a fixed step, gauges, snapshots, cross section
    ("soliton", {"amplitude": 0.2}, 256, 4, 0.0, 0.6, 2e-3, [(10.0, 0.0), (-3.3, 1.0)], [0.0, 0.301, 0.6], 3, 0.0),
    # fully reflecting 2D obstacle, clamped gauges
    ("gaussian_obstacle", {"bounded": 1}, 61, 31, 0.0, 0.3, 2.5e-3, [(0.0, 0.0), (50.0, 50.0)], [0.1, 0.3], 5, 1.0),
    # wall in x, periodic y; the scenario's own gauge and (empty) snapshot list
    ("wall_reflection", {}, 101, 4, 0.0, 1.0, 4e-3, None, None, 1, None),
    # manufactured forcing (device source terms: tolerance-level, not bitwise)
    ("manufactured", {}, 32, 32, 0.0, 0.05, 5e-4, [(0.25, 0.5)], [0.05], 4, None),
]


@pytest.mark.parametrize("name,params,nx,ny,t0,tf,dt,gauges,snaps,stride,xsec", RUN_CASES)
def test_cli_run_fixed_step_matches_reference(tmp_path, name, params, nx, ny, t0, tf, dt, gauges, snaps, stride,
                                              xsec):
    text = f"[run]\nscenario = {name}\nnx = {nx}\nny = {ny}\nt_final = {tf!r}\n"
    text += "[scenario]\n" + "".join(f"{k} = {v!r}\n" for k, v in params.items())
    text += f"[integrator]\nfixed_dt = {dt!r}\n[output]\nconservation_stride = {stride}\n"
    if gauges is not None:
        text += "gauges = " + "; ".join(f"{x!r}, {y!r}" for x, y in gauges) + "\n"
    if snaps is not None:
        text += "snapshot_times = " + ", ".join(repr(s) for s in snaps) + "\n"
    if xsec is not None:
        text += f"cross_section_y = {xsec!r}\n"
    ddir = str(tmp_path / "dev")
    assert cli.main(["run", "--config", _write_cfg(tmp_path, text), "--output", ddir]) == 0

    spec = S.make_scenario(name, params)
    orc = Oracle("ref")
    orc.set_threads(8)
    g, ph, b, q0, sk, _, _ = orc.prepare(name, nx, ny, **params)
    rdir = str(tmp_path / "ref")
    gz = gauges if gauges is not None else spec.gauges
    tg = snaps if snaps is not None else spec.snapshot_times
    qr, rr = orc.run_recorded(g, ph, b, q0, t0, tf, default_cfg(fixed_dt=dt), rdir, gauges=gz, targets=tg,
                              stride=stride, source_kind=sk)
    meta = json.loads(_read(os.path.join(ddir, "run_meta.json")))
    assert meta["status"] == "ok" and not rr.aborted
    assert (meta["steps"]["accepted"], meta["steps"]["rejected"], meta["steps"]["rhs_evals"]) == (
        rr.accepted, rr.rejected, rr.rhs_evals)
    assert meta["time"]["t_reached"] == rr.t
    bitwise = not spec.has_source
    ref_files = sorted(f for f in os.listdir(rdir) if f.endswith(".csv"))
    dev_files = sorted(f for f in os.listdir(ddir) if f.endswith(".csv") and f != "cross_section.csv")
    assert dev_files == ref_files
    for f in ref_files:
        if f == "conservation.csv":
            a, r = _table(os.path.join(ddir, f)), _table(os.path.join(rdir, f))
            assert a.shape == r.shape and np.array_equal(a[:, 0], r[:, 0])
            assert np.allclose(a[:, 1:3], r[:, 1:3], rtol=1e-13, atol=0)
            assert np.all(np.abs(a[:, 3] - r[:, 3]) <= 1e-10 * np.abs(r[:, 2]))
        elif bitwise:
            assert _read(os.path.join(ddir, f)) == _read(os.path.join(rdir, f)), f
        else:
            a, r = _table(os.path.join(ddir, f)), _table(os.path.join(rdir, f))
            assert a.shape == r.shape and np.allclose(a, r, rtol=1e-11, atol=1e-13), f
    if xsec is not None:
        grid = spec.grid(nx, ny)
        want = tmp_path / "xsec.csv"
        R.write_cross_section_csv(str(want), grid, qr, b, xsec)
        assert _read(os.path.join(ddir, "cross_section.csv")) == _read(want)
    assert meta["conservation"]["mass_initial"] > 0 and abs(meta["conservation"]["mass_drift_rel"]) < 1e-12 or \
        spec.has_source


def test_cli_run_adaptive_matches_reference(tmp_path):
    text = ("[run]\nscenario = lake_at_rest\nnx = 40\nny = 36\nt_final = 0.05\n[scenario]\nbounded = 1\n"
            "bump_amplitude = 0.3\n[integrator]\nabs_tol = 1e-7\nrel_tol = 1e-7\n[output]\n"
            "gauges = 0.5, 0.5\nsnapshot_times = 0.05\n")
    ddir = str(tmp_path / "dev")
    assert cli.main(["run", "--config", _write_cfg(tmp_path, text), "--output", ddir]) == 0
    orc = Oracle("ref")
    orc.set_threads(8)
    g, ph, b, q0, sk, *_ = orc.prepare("lake_at_rest", 40, 36, bounded=1, bump_amplitude=0.3)
    # a state at rest stays at rest: perturb nothing, compare counts and values
    qr, rr = orc.run_recorded(g, ph, b, q0, 0.0, 0.05, default_cfg(abs_tol=1e-7, rel_tol=1e-7),
                              str(tmp_path / "ref"), gauges=[(0.5, 0.5)], targets=[0.05])
    meta = json.loads(_read(os.path.join(ddir, "run_meta.json")))
    assert (meta["steps"]["accepted"], meta["steps"]["rejected"]) == (rr.accepted, rr.rejected)
    a, r = _table(os.path.join(ddir, "gauges.csv")), _table(str(tmp_path / "ref" / "gauges.csv"))
    assert a.shape == r.shape and np.allclose(a, r, rtol=1e-12, atol=1e-14)


def test_cli_converge_matches_reference(tmp_path):
    res = [16, 32, 64]
    text = ("[run]\nscenario = manufactured\nt_final = 0.25\n[converge]\nresolutions = "
            + ", ".join(map(str, res)) + "\n")
    ddir = str(tmp_path / "dev")
    assert cli.main(["converge", "--config", _write_cfg(tmp_path, text), "--output", ddir]) == 0
    rows = _read(os.path.join(ddir, "convergence.csv")).splitlines()
    assert rows[0] == "nx,dx,err_h,eoc_h,err_u,eoc_u,err_v,eoc_v,err_w,eoc_w,err_eta,eoc_eta,status"
    tab = [r.split(",") for r in rows[1:]]
    assert [int(r[0]) for r in tab] == res and all(r[-1] == "ok" for r in tab)
    # reference: the same rungs through its own adaptive_solve at tol 1e-10
    orc = Oracle("ref")
    orc.set_threads(8)
    fn = orc.lib.ref_mms_exact_field
    fn.restype = None
    import ctypes as C
    for k, n in enumerate(res):
        g, ph, b, q0, sk, *_ = orc.prepare("manufactured", n, n)
        q, rec = orc.solve(g, ph, b, q0, 0.0, 0.25, default_cfg(abs_tol=1e-10, rel_tol=1e-10), source_kind=sk)
        ex = np.empty_like(q)
        fn(C.byref(g), C.c_double(rec.t), ex.ctypes.data_as(C.POINTER(C.c_double)))
        m = n * n
        for v in range(5):
            err = orc.discrete_l2_error(g, q[v * m:(v + 1) * m], ex[v * m:(v + 1) * m])
            mine = float(tab[k][2 + 2 * v])
            assert abs(mine - err) <= 1e-7 * err, (n, v, mine, err)
    eocs = [float(x) for x in tab[-1][3:-1:2]]
    assert all(1.8 <= e <= 2.2 for e in eocs), eocs
    meta = json.loads(_read(os.path.join(ddir, "run_meta.json")))
    assert meta["status"] == "ok" and meta["resolutions"] == res and meta["integrator"]["abs_tol"] == 1e-10


def test_cli_bench_and_errors(tmp_path, capsys):
    text = "[bench]\nresolutions = 32, 64\nrepetitions = 3\nwarmups = 1\n"
    ddir = str(tmp_path / "bench")
    assert cli.main(["bench", "--config", _write_cfg(tmp_path, text), "--output", ddir]) == 0
    rows = _read(os.path.join(ddir, "bench.csv")).splitlines()
    assert rows[0] == "nx,ny,n_total,seconds_per_rhs,seconds_per_rhs_min,threads" and len(rows) == 3
    assert rows[1].startswith("32,32,1024,") and rows[2].startswith("64,64,4096,")
    meta = json.loads(_read(os.path.join(ddir, "run_meta.json")))
    assert meta["command"] == "bench" and meta["scenario"]["name"] == "still_water" and len(meta["rungs"]) == 2
    # configuration errors exit 2 with the reference message
    bad = tmp_path / "bad.cfg"
    bad.write_text("[run]\nscenario = soliton\n[scenario]\namplitud = 0.1\n")
    assert cli.main(["run", "--config", str(bad), "--output", str(tmp_path / "x")]) == 2
    assert "scenario 'soliton': unknown parameter 'amplitud'" in capsys.readouterr().err
    bad.write_text("[run]\nnx = many\n")
    assert cli.main(["run", "--config", str(bad)]) == 2
    bad.write_text("[run]\nscenario = favre\n[converge]\nresolutions = 8, 16\n")
    assert cli.main(["converge", "--config", str(bad)]) == 2
    assert "has no exact solution" in capsys.readouterr().err


def test_cli_run_abort_exit_code(tmp_path):
    """A solver abort (fixed step into a dry node) exits 1 with the reason in run_meta.json."""
    text = ("[run]\nscenario = still_water\nnx = 16\nny = 16\nt_final = 1\n[scenario]\ndepth = 1e-13\n"
            "[integrator]\nfixed_dt = 0.01\n")
    ddir = str(tmp_path / "dev")
    rc = cli.main(["run", "--config", _write_cfg(tmp_path, text), "--output", ddir])
    meta = json.loads(_read(os.path.join(ddir, "run_meta.json")))
    assert rc == 1 and meta["status"] == "aborted" and "depth" in meta["abort_reason"]


# ------------------------------------------------------------------ the reference's test_cli.cpp cases

def _cfg(**kw):
    from paper_2601_02540_b200.config import RunConfig
    c = RunConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_ref_cli_run_full_output_set(tmp_path):
    """test_cli.cpp:62-132"""
    d = str(tmp_path / "run_lake")
    cfg = _cfg(scenario="lake_at_rest", nx=20, ny=20, t_final=1.0, output_dir=d, gauges_set=True,
               gauges=[(0.0, 0.0)], snapshots_set=True, snapshot_times=[0.0, 0.5], cross_section_set=True,
               cross_section_y=0.0)
    assert cli.cmd_run(cfg, open(os.devnull, "w")) == 0
    for f in ("conservation.csv", "gauges.csv", "run_meta.json", "cross_section.csv", "snapshot_t0.csv",
              "snapshot_t0.5.csv"):
        assert os.path.exists(os.path.join(d, f)), f
    assert _read(os.path.join(d, "conservation.csv")).splitlines()[0] == \
        "t,total_mass,total_energy,semidiscrete_energy_rate"
    cons = _table(os.path.join(d, "conservation.csv"))
    assert len(cons) >= 2
    m0, e0 = cons[0, 1], cons[0, 2]
    assert np.all(np.abs(cons[:, 1] - m0) <= 1e-12 * abs(m0))
    assert np.all(np.abs(cons[:, 2] - e0) <= 1e-12 * abs(e0))
    assert np.all(np.abs(cons[:, 3]) <= 1e-11 * abs(e0))
    g = _table(os.path.join(d, "gauges.csv"))
    assert [ln for ln in _read(os.path.join(d, "gauges.csv")).splitlines() if not ln.startswith("#")][0] == \
        "t,gauge_1"
    assert np.all(np.abs(g[:, 1] - 1.0) <= 1e-12)
    meta = json.loads(_read(os.path.join(d, "run_meta.json")))
    assert meta["status"] == "ok" and meta["command"] == "run" and meta["scenario"]["name"] == "lake_at_rest"
    assert meta["grid"]["nx"] == 20 and meta["grid"]["boundary_x"] == "periodic"
    assert meta["time"]["t_reached"] == 1.0
    st = meta["steps"]
    assert st["rhs_evals"] == 3 * (st["accepted"] + st["rejected"]) + 1 + st["rhs_evals_setup"]
    assert abs(meta["conservation"]["mass_drift_rel"]) <= 1e-12
    assert len(meta["snapshots"]) == 2 and meta["snapshots"][0]["target"] == 0.0
    assert meta["snapshots"][0]["file"] == "snapshot_t0.csv"
    snap = _read(os.path.join(d, "snapshot_t0.5.csv")).splitlines()
    assert snap[0] == "x,y,h,u,v,w,eta,b" and len(snap) == 1 + 20 * 20


def test_ref_cli_reruns_byte_identical(tmp_path):
    """test_cli.cpp:134-156 (adaptive run: the device sums are deterministic)."""
    dirs = []
    for name in ("rerun_a", "rerun_b"):
        d = str(tmp_path / name)
        cfg = _cfg(scenario="lake_at_rest", nx=16, ny=16, t_final=0.5, output_dir=d, gauges_set=True,
                   gauges=[(1.0, -1.0)], snapshots_set=True, snapshot_times=[0.25])
        assert cli.cmd_run(cfg, open(os.devnull, "w")) == 0
        dirs.append(d)
    for f in ("conservation.csv", "gauges.csv", "snapshot_t0.25.csv"):
        assert _read(os.path.join(dirs[0], f)) == _read(os.path.join(dirs[1], f))


def test_ref_cli_abort_partial_record(tmp_path):
    """test_cli.cpp:158-178"""
    d = str(tmp_path / "run_abort")
    cfg = _cfg(scenario="lake_at_rest", nx=16, ny=16, t_final=5.0, output_dir=d)
    cfg.integrator.max_steps = 1
    assert cli.cmd_run(cfg, open(os.devnull, "w")) == 1
    meta = json.loads(_read(os.path.join(d, "run_meta.json")))
    assert meta["status"] == "aborted" and "step budget" in meta["abort_reason"]
    assert meta["time"]["t_reached"] < 5.0
    assert len(_table(os.path.join(d, "conservation.csv"))) >= 1


def test_ref_cli_unknown_scenario_touches_no_disk(tmp_path):
    """test_cli.cpp:180-187"""
    d = str(tmp_path / "should_not_exist")
    with pytest.raises(ValueError):
        cli.cmd_run(_cfg(scenario="maelstrom", output_dir=d), open(os.devnull, "w"))
    assert not os.path.exists(d)


def test_ref_cli_converge_ladder(tmp_path):
    """test_cli.cpp:189-228"""
    d = str(tmp_path / "converge_mms")
    cfg = _cfg(scenario="manufactured", t_final=0.5, resolutions=[16, 32], tolerances_set=True, output_dir=d)
    cfg.integrator.abs_tol = 1e-8
    cfg.integrator.rel_tol = 1e-8
    assert cli.cmd_converge(cfg, open(os.devnull, "w")) == 0
    rows = _read(os.path.join(d, "convergence.csv")).splitlines()
    head = rows[0].split(",")
    assert len(head) == 2 + 2 * 5 + 1 and head[:3] == ["nx", "dx", "err_h"] and head[-1] == "status"
    t = [r.split(",") for r in rows[1:]]
    assert len(t) == 2 and float(t[0][0]) == 16.0 and float(t[1][0]) == 32.0
    assert float(t[1][2]) < float(t[0][2])
    meta = json.loads(_read(os.path.join(d, "run_meta.json")))
    assert meta["status"] == "ok" and meta["row_status"][0] == "ok"
    bad = _cfg(**{**vars(cfg), "scenario": "still_water"})
    with pytest.raises(ValueError, match="no exact solution"):
        cli.cmd_converge(bad, open(os.devnull, "w"))
    bad = _cfg(**{**vars(cfg), "resolutions": [8]})
    with pytest.raises(ValueError, match=">= 2"):
        cli.cmd_converge(bad, open(os.devnull, "w"))


def test_ref_cli_bench_ladder(tmp_path):
    """test_cli.cpp:230-266"""
    d = str(tmp_path / "bench_small")
    cfg = _cfg(bench_resolutions=[4, 6, 8], bench_repetitions=3, bench_warmups=1, output_dir=d)
    assert cli.cmd_bench(cfg, open(os.devnull, "w")) == 0
    rows = _read(os.path.join(d, "bench.csv")).splitlines()
    assert rows[0].split(",") == ["nx", "ny", "n_total", "seconds_per_rhs", "seconds_per_rhs_min", "threads"]
    assert len(rows) == 4
    for r in rows[1:]:
        v = [float(x) for x in r.split(",")]
        assert v[2] == v[0] * v[1] and v[3] > 0 and v[4] > 0 and v[4] <= v[3]
    bad_dir = str(tmp_path / "bench_bad")
    with pytest.raises(ValueError, match="4-node minimum"):
        cli.cmd_bench(_cfg(**{**vars(cfg), "bench_resolutions": [2, 4], "output_dir": bad_dir}),
                      open(os.devnull, "w"))
    assert not os.path.exists(bad_dir)
    with pytest.raises(ValueError, match="repetitions"):
        cli.cmd_bench(_cfg(**{**vars(cfg), "bench_repetitions": 0}), open(os.devnull, "w"))
