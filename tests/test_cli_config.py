"""CLI front end, host side: the configuration parser
(config.hpp) and the scenario registry (scenarios.hpp), no GPU.

* config.py is checked differentially against the reference's own
  parse_config_text (oracle/_ref ref_parse_config) on the reference's example
  configurations, the cases of its test_config.cpp and a seeded random corpus
  of well- and ill-formed files: same fields, or the same error message.
* The native scenario registry (hsgn_scenarios.cpp) must sample b, h, u, v
  bit-identically to the reference's make_scenario + prepare_run for every
  scenario (oracle/_ref ref_prepare), with the same domain / physics / time
  metadata and the same error messages.
"""
import ctypes as C
import glob
import math
import os
import random

import numpy as np
import pytest

from oracle_lib import Oracle, make_grid as omake_grid, ref_available

from paper_2601_02540_b200 import config as CF
from paper_2601_02540_b200 import scenarios as S

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
REF_CONFIGS = sorted(glob.glob("/root/reference/proj/configs/*.cfg"))


def _dump(c: CF.RunConfig) -> str:
    """The canonical field dump of ref_parse_config for a Python RunConfig."""
    lines = []

    def num(k, v):
        lines.append(f"{k}={'%.17g' % float(v)}")
    lines.append(f"scenario={c.scenario}")
    for k in sorted(c.scenario_params):
        num("param." + k, c.scenario_params[k])
    for k in ("nx", "ny", "t0", "t_final", "threads"):
        num(k, getattr(c, k))
    ic = c.integrator
    for k in ("abs_tol", "rel_tol", "dt_initial", "dt_max", "fixed_dt", "max_steps", "safety", "growth_cap",
              "shrink_floor"):
        num(k, getattr(ic, k))
    num("tolerances_set", c.tolerances_set)
    lines.append(f"output_dir={c.output_dir}")
    num("gauges_set", c.gauges_set)
    for x, y in c.gauges:
        num("gauge.x", x)
        num("gauge.y", y)
    num("snapshots_set", c.snapshots_set)
    for t in c.snapshot_times:
        num("snapshot", t)
    num("conservation_stride", c.conservation_stride)
    num("cross_section_set", c.cross_section_set)
    num("cross_section_y", c.cross_section_y)
    for r in c.resolutions:
        num("resolution", r)
    num("converge_ny", c.converge_ny)
    for r in c.bench_resolutions:
        num("bench_resolution", r)
    num("bench_repetitions", c.bench_repetitions)
    num("bench_warmups", c.bench_warmups)
    return "\n".join(lines) + "\n"


def _ref_parse(text: str):
    lib = Oracle("ref").lib
    fn = lib.ref_parse_config
    fn.restype = C.c_int
    fn.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
    buf = C.create_string_buffer(1 << 16)
    st = fn(text.encode(), buf, len(buf))
    return st, buf.value.decode()


def _mine(text: str):
    try:
        return 0, _dump(CF.parse_config_text(text))
    except CF.ConfigError as e:
        return -1, str(e)


ROUND_TRIP = """# solver configuration
[run]
scenario = soliton
nx = 400
ny = 4
t_final = 2.5
threads = 2

[scenario]
amplitude = 0.1
half_length = 30

[integrator]
abs_tol = 1e-9
rel_tol = 1e-9
dt_max = 0.5

[output]
directory = results/soliton
gauges = 0, 0; 1.5, -2.25
snapshot_times = 0.5, 1.0, 2.5
conservation_stride = 10
cross_section_y = 0.25

[converge]
resolutions = 100, 200, 400
ny = 4

[bench]
resolutions = 32, 48, 64, 96
repetitions = 7
warmups = 2
"""

ERRORS = ["[run]\nscenario = x\nnz = 4\n", "[rnu]\n", "[run]\nscenario soliton\n", "scenario = x\n", "[run\n",
          "[run]\nnx = many\n", "[run]\nnx = 2.5\n", "[output]\ngauges = 1.0; 2.0, 3.0\n",
          "[output]\nconservation_stride = 0\n", "[scenario]\namplitude = big\n", "[run]\n = 3\n",
          "[output]\ngauges = ;\n", "[output]\nsnapshot_times = , ,\n", "[converge]\nresolutions = 1, 2.5\n",
          "[integrator]\nmax_steps = 1e3\nfixed_dt = 0x1p-10\n", "[integrator]\ndt_max = inf\n",
          "[run]\nt0 = nan\nnx = -0\n", "[bench]\nresolutions = 8,\n", "  # c\n\t[run]\t\r\nscenario =\n"]


def test_config_round_trip_fields():
    """test_config.cpp:32-95, 97-112 (the same expectations, Python side)."""
    c = CF.parse_config_text(ROUND_TRIP)
    assert (c.scenario, c.nx, c.ny, c.t_final, c.threads) == ("soliton", 400, 4, 2.5, 2)
    assert math.isnan(c.t0)
    assert c.scenario_params == {"amplitude": 0.1, "half_length": 30.0}
    assert (c.integrator.abs_tol, c.integrator.rel_tol, c.integrator.dt_max, c.tolerances_set) == (1e-9, 1e-9,
                                                                                                   0.5, True)
    assert c.output_dir == "results/soliton" and c.gauges == [(0.0, 0.0), (1.5, -2.25)] and c.gauges_set
    assert c.snapshot_times == [0.5, 1.0, 2.5] and c.snapshots_set and c.conservation_stride == 10
    assert c.cross_section_set and c.cross_section_y == 0.25
    assert c.resolutions == [100, 200, 400] and c.converge_ny == 4
    assert (c.bench_resolutions, c.bench_repetitions, c.bench_warmups) == ([32, 48, 64, 96], 7, 2)
    d = CF.parse_config_text("")
    assert d.scenario == "" and d.nx == 0 and not d.tolerances_set and d.output_dir == "out"
    assert d.bench_resolutions == [128, 181, 256, 362, 512] and (d.bench_repetitions, d.bench_warmups) == (50, 5)


def test_config_errors_and_precedence(tmp_path, monkeypatch):
    """test_config.cpp:114-201."""
    with pytest.raises(CF.ConfigError, match="line 3.*nz"):
        CF.parse_config_text("[run]\nscenario = x\nnz = 4\n")
    with pytest.raises(CF.ConfigError, match="cannot open"):
        CF.parse_config_file("/nonexistent/path.cfg")
    assert CF.parse_config_text("# leading comment\n\n  [run]  \n   scenario   =   favre   \n\n# done\n").scenario \
        == "favre"
    monkeypatch.setenv("THREADS", "3")
    c = CF.parse_config_text("")
    CF.apply_thread_env(c)
    assert c.threads == 3
    monkeypatch.setenv("THREADS", "8")
    c = CF.parse_config_text("[run]\nthreads = 2\n")
    CF.apply_thread_env(c)
    assert c.threads == 2
    monkeypatch.setenv("THREADS", "lots")
    with pytest.raises(CF.ConfigError, match="THREADS"):
        CF.apply_thread_env(CF.parse_config_text(""))


def _corpus(seed=20261018, n=300):
    rng = random.Random(seed)
    keys = {s: sorted(k) for s, k in CF._SCHEMA.items()}
    keys["scenario"] = ["amplitude", "h_inf", "bounded", "lambda"]
    vals = ["1", "2.5", "-3", "1e-3", "0x1.8p1", "  7  ", "abc", "1,2", "3, 4; 5, 6", "0", "-0", "1e400", "inf",
            "nan", "", "4, 8, 16", "1.0; 2.0", ".5", "5.", "+2", "1_0", "results/x y"]
    out = []
    for _ in range(n):
        lines = []
        for _ in range(rng.randint(1, 8)):
            r = rng.random()
            if r < 0.15:
                lines.append("[" + rng.choice(list(keys) + ["bogus"]) + "]")
            elif r < 0.2:
                lines.append(rng.choice(["# comment", "", "   ", "[run", "novalue", "= 3"]))
            else:
                sec = rng.choice(list(keys))
                lines.append(f"[{sec}]")
                lines.append(f"{rng.choice(keys[sec] + ['zz'])} = {rng.choice(vals)}")
        out.append("\n".join(lines) + "\n")
    return out


@needs_ref
def test_config_parser_matches_reference_differential():
    texts = [ROUND_TRIP, ""] + ERRORS + _corpus()
    for path in REF_CONFIGS:
        with open(path) as fh:
            texts.append(fh.read())
    assert len(REF_CONFIGS) >= 10 or not os.path.isdir("/root/reference")
    for text in texts:
        assert _mine(text) == _ref_parse(text), text


# ------------------------------------------------------------------ scenarios

SCENARIO_CASES = [("soliton", {}), ("soliton", {"axis": 1, "direction": -1, "amplitude": 0.3, "center": 2.5}),
                  ("manufactured", {}), ("manufactured", {"bounded": 1, "lambda": 40}),
                  ("dingemans", {}), ("dingemans", {"wave_period": 1.5, "n_waves": 3, "x_offset": 5}),
                  ("head_on_collision", {}), ("wall_reflection", {}), ("wall_reflection", {"amplitude": 0.65}),
                  ("gaussian_obstacle", {}), ("gaussian_obstacle", {"bounded": 1}), ("riemann", {}),
                  ("favre", {"eps": 0.2, "alpha": 0.5}), ("still_water", {"depth": 2}),
                  ("lake_at_rest", {"bounded": 1, "bump_width": 0.7})]


@needs_ref
@pytest.mark.parametrize("name,params", SCENARIO_CASES)
def test_scenario_initial_data_bitwise(name, params):
    orc = Oracle("ref")
    spec = S.make_scenario(name, params)
    for nx, ny in [(min(spec.nx_default, 400), max(4, min(spec.ny_default, 64))), (37, 5)]:
        g, ph, b, q0, sk, t0, tf = orc.prepare(name, nx, ny, **params)
        bb, q = S.sample_initial(spec, nx, ny)
        n = nx * ny
        assert np.array_equal(bb, b)
        assert np.array_equal(q[:3 * n], q0[:3 * n])
    assert (spec.x_min, spec.x_max, spec.y_min, spec.y_max) == (g.x_min, g.x_max, g.y_min, g.y_max)
    assert (int(spec.kind_x), int(spec.kind_y), spec.g, spec.lambda_) == (g.kind_x, g.kind_y, ph.g, ph.lambda_)
    assert (int(spec.has_source), spec.t0, spec.t_final) == (sk, t0, tf)
    g0 = orc.prepare(name, 0, 0, **params)[0]
    assert (spec.nx_default, spec.ny_default) == (g0.nx, g0.ny)


@needs_ref
def test_scenario_full_default_grids_bitwise():
    """The 1D-profile scenarios at their default resolutions (dingemans 3680 x 4 ...)."""
    orc = Oracle("ref")
    for name in ("dingemans", "riemann", "favre", "wall_reflection", "head_on_collision"):
        spec = S.make_scenario(name)
        g, ph, b, q0, *_ = orc.prepare(name)
        bb, q = S.sample_initial(spec, spec.nx_default, spec.ny_default)
        n = g.nx * g.ny
        assert np.array_equal(bb, b) and np.array_equal(q[:3 * n], q0[:3 * n]), name


@needs_ref
def test_scenario_errors_match_reference():
    orc = Oracle("ref")
    for name, params in [("nosuch", {}), ("soliton", {"amplitud": 1.0}), ("soliton", {"amplitude": -1.0}),
                         ("head_on_collision", {"h_inf": 0.0}), ("lake_at_rest", {"center": 1.0})]:
        with pytest.raises(ValueError) as mine:
            S.make_scenario(name, params)
        with pytest.raises(ValueError) as ref:
            orc.prepare(name, 8, 8, **params)
        assert str(mine.value) == str(ref.value)


def test_scenario_registry_metadata():
    """scenarios.hpp:700-705 names; defaults that the CLI relies on."""
    assert S.scenario_names() == ["soliton", "manufactured", "dingemans", "head_on_collision", "wall_reflection",
                                  "gaussian_obstacle", "riemann", "favre", "still_water", "lake_at_rest"]
    s = S.make_scenario("soliton")
    assert s.exact_vars == ["h", "u"] and s.lambda_ == 30000.0 and (s.nx_default, s.ny_default) == (200, 4)
    assert S.make_scenario("soliton", {"axis": 1}).exact_vars == ["h", "v"]
    m = S.make_scenario("manufactured")
    assert m.has_source and m.exact_vars == ["h", "u", "v", "w", "eta"]
    d = S.make_scenario("dingemans")
    assert len(d.gauges) == 6 and d.gauges[0] == (3.04, -46.0)
    assert not S.make_scenario("favre").has_exact


@needs_ref
def test_exact_solutions():
    """manufactured: the hand-derived closed form against the reference's
    generated exact_state (ref_mms_exact_field) to round-off; soliton: the
    translated profile at t = 0 equals the initial data bit for bit."""
    spec = S.make_scenario("manufactured")
    fn = Oracle("ref").lib.ref_mms_exact_field
    fn.restype = None
    for t in (0.0, 0.37, 1.0):
        mine = S.exact_state(spec, 40, 36, t)
        q = np.empty(5 * 40 * 36)
        fn(C.byref(omake_grid(40, 36)), C.c_double(t), q.ctypes.data_as(C.POINTER(C.c_double)))
        assert np.max(np.abs(mine - q)) <= 1e-14 * np.max(np.abs(q))
    sol = S.make_scenario("soliton", {"center": 3.0, "direction": -1})
    b, q = S.sample_initial(sol, 200, 4)
    ex = S.exact_state(sol, 200, 4, 0.0)
    x = np.tile(-30.0 + np.arange(200) * 0.3, 4)
    keep = np.abs(x - 3.0) < 30.0  # nodes the periodic wrap leaves in place
    for f in (0, 1):
        assert np.array_equal(ex[f * 800:(f + 1) * 800][keep], q[f * 800:(f + 1) * 800][keep])
    assert np.array_equal(ex[4 * 800:], ex[:800])
    # one traversal later the profile is back (periodic translation)
    ex1 = S.exact_state(sol, 200, 4, sol.t_final)
    assert np.max(np.abs(ex1[:800] - q[:800])[keep]) < 1e-12
