"""ctypes loaders for the two CPU checkers under oracle/ -- TEST INFRASTRUCTURE.

* ``Oracle("orc")`` -> oracle/liboracle.so, the from-scratch C restatement
  (oracle/hsgn_oracle.c).  Rebuilt with ``make -C oracle oracle`` if absent
  (gcc is in the image on the GPU box too).
* ``Oracle("ref")`` -> oracle/_ref/libhsgn_ref.so, the unmodified reference
  headers compiled in place (oracle/ref_capi.cpp).  Only present where
  /root/reference existed at build time; callers skip when it is missing.

Both export the same function names with prefixes ``orc_`` / ``ref_`` and the
structs of oracle/oracle_abi.h, so tests can run one check against either.
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORC_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libhsgn_ref.so")

D = C.c_double
PD = C.POINTER(C.c_double)
I64 = C.c_int64


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("kind_x", C.c_int32), ("kind_y", C.c_int32),
                ("x_min", D), ("x_max", D), ("y_min", D), ("y_max", D)]


class Phys(C.Structure):
    _fields_ = [("g", D), ("lambda_", D), ("h_floor", D)]


class Cfg(C.Structure):
    _fields_ = [("abs_tol", D), ("rel_tol", D), ("dt_initial", D), ("dt_max", D), ("safety", D),
                ("growth_cap", D), ("shrink_floor", D), ("max_steps", I64), ("fixed_dt", D),
                ("h_floor", D)]


class Record(C.Structure):
    _fields_ = [("t", D), ("accepted", I64), ("rejected", I64), ("rhs_evals", I64),
                ("rhs_evals_setup", I64), ("aborted", C.c_int32), ("reason", C.c_char * 256)]


def default_cfg(**kw) -> Cfg:
    """reference time_integration.hpp:18-29 defaults."""
    c = Cfg(1e-6, 1e-6, 0.0, float("inf"), 0.9, 5.0, 0.2, 50_000_000, 0.0, 1e-12)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def make_grid(nx, ny, x_min=-1.0, x_max=1.0, y_min=-1.0, y_max=1.0, kind_x=0, kind_y=0) -> Grid:
    return Grid(nx, ny, int(kind_x), int(kind_y), x_min, x_max, y_min, y_max)


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(PD)


def ensure_built() -> None:
    if not os.path.exists(ORC_SO):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, "oracle"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Oracle:
    def __init__(self, which: str = "orc"):
        self.which = which
        if which == "orc":
            ensure_built()
            self.lib = C.CDLL(ORC_SO)
        elif which == "ref":
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(REF_SO)
            self.lib = C.CDLL(REF_SO)
        else:
            raise ValueError(which)
        pre = which + "_"
        L = self.lib

        def f(name, res, *args):
            fn = getattr(L, pre + name)
            fn.restype = res
            fn.argtypes = list(args)
            return fn

        G, PH = C.POINTER(Grid), C.POINTER(Phys)
        self._rhs = f("rhs", C.c_int, G, PH, PD, C.c_int, C.c_int, D, PD, PD, C.POINTER(I64))
        self._solve = (f("solve", C.c_int, G, PH, PD, C.c_int, PD, D, D, C.POINTER(Cfg), PD,
                         C.POINTER(Record)) if which == "orc" else
                       f("solve", C.c_int, G, PH, PD, C.c_int, PD, D, D, C.POINTER(Cfg), PD,
                         C.POINTER(Record), PD, I64, C.POINTER(I64)))
        self._mass = f("total_mass", D, G, PD)
        self._energy = f("total_energy", D, G, PH, PD, PD)
        self._rate = f("energy_rate", D, G, PH, PD, PD, PD)
        self._mws = f("mass_weighted_sum", D, G, PD)
        self._l2 = f("discrete_l2_error", D, G, PD, PD)
        self._init_aux = f("init_auxiliary", None, G, PD, PD)
        self._apply_d = f("apply_d", None, G, C.c_int, PD, PD)
        self._sat = f("sat", None, G, PD, PD, PD)
        self._errn = f("error_norm", D, D, G, PD, PD, PD, PD, PD, PD, D, D, PD)
        self._sbp = f("check_sbp", C.c_int, C.c_int, C.c_int, D, PD)
        self._bath = f("mms_bathymetry", D, D, D)
        self._mstate = f("mms_state", None, D, D, D, PD)
        self._mstate_dt = f("mms_state_dt", None, D, D, D, PD)
        self._msrc = f("mms_source", None, D, D, D, D, PD)
        self._threads = f("set_threads", None, C.c_int)
        if which == "ref":
            self._prepare = f("prepare", C.c_int, C.c_char_p, C.POINTER(C.c_char_p), PD, C.c_int,
                              C.c_int, C.c_int, G, PH, PD, PD, C.POINTER(C.c_int), PD, PD,
                              C.c_char_p, C.c_int)
            self._rhs_repeat = f("rhs_repeat", C.c_int, G, PH, PD, D, PD, PD, C.c_int)
            self._run_rec = f("run_recorded", C.c_int, G, PH, PD, C.c_int, PD, D, D, C.POINTER(Cfg), PD,
                              C.POINTER(Record), C.c_char_p, C.c_int, PD, C.c_int, PD, I64)
        else:
            self._fixed = f("bs3_fixed_steps", C.c_int, G, PH, PD, PD, PD, D, D, C.c_int, C.c_int)

    # ------------------------------------------------------------------ API
    def set_threads(self, n: int) -> None:
        self._threads(int(n))

    def rhs(self, grid: Grid, phys: Phys, b, q, t=0.0, source_kind=0, variant=0, out=None):
        """Returns (status, out, n_evals); status 1 = depth_error (out untouched)."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros_like(q) if out is None else out
        ne = I64(0)
        st = self._rhs(C.byref(grid), C.byref(phys), _p(np.ascontiguousarray(b, np.float64)),
                       source_kind, variant, t, _p(q), _p(out), C.byref(ne))
        return st, out, ne.value

    def solve(self, grid, phys, b, q0, t0, t_final, cfg, source_kind=0):
        q0 = np.ascontiguousarray(q0, dtype=np.float64)
        out = np.empty_like(q0)
        rec = Record()
        args = [C.byref(grid), C.byref(phys), _p(np.ascontiguousarray(b, np.float64)), source_kind,
                _p(q0), t0, t_final, C.byref(cfg), _p(out), C.byref(rec)]
        if self.which == "ref":
            args += [None, 0, None]
        self._solve(*args)
        return out, rec

    def total_mass(self, grid, q):
        return self._mass(C.byref(grid), _p(np.ascontiguousarray(q, np.float64)))

    def total_energy(self, grid, phys, b, q):
        return self._energy(C.byref(grid), C.byref(phys), _p(np.ascontiguousarray(b, np.float64)),
                            _p(np.ascontiguousarray(q, np.float64)))

    def energy_rate(self, grid, phys, b, q, qt):
        return self._rate(C.byref(grid), C.byref(phys), _p(np.ascontiguousarray(b, np.float64)),
                          _p(np.ascontiguousarray(q, np.float64)), _p(np.ascontiguousarray(qt, np.float64)))

    def mass_weighted_sum(self, grid, f):
        return self._mws(C.byref(grid), _p(np.ascontiguousarray(f, np.float64)))

    def discrete_l2_error(self, grid, a, b):
        return self._l2(C.byref(grid), _p(np.ascontiguousarray(a, np.float64)),
                        _p(np.ascontiguousarray(b, np.float64)))

    def init_auxiliary(self, grid, b, q):
        q = np.array(q, dtype=np.float64, copy=True)
        self._init_aux(C.byref(grid), _p(np.ascontiguousarray(b, np.float64)), _p(q))
        return q

    def apply_d(self, grid, direction, u):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty_like(u)
        self._apply_d(C.byref(grid), direction, _p(u), _p(out))
        return out

    def sat(self, grid, hu, hv):
        hu = np.ascontiguousarray(hu, np.float64)
        out = np.zeros_like(hu)
        self._sat(C.byref(grid), _p(hu), _p(np.ascontiguousarray(hv, np.float64)), _p(out))
        return out

    def error_norm(self, dt, grid, k1, k2, k3, k4, y, ynew, atol, rtol):
        mh = D(0.0)
        arrs = [np.ascontiguousarray(a, np.float64) for a in (k1, k2, k3, k4, y, ynew)]
        e = self._errn(dt, C.byref(grid), *[_p(a) for a in arrs], atol, rtol, C.byref(mh))
        return e, mh.value

    def check_sbp(self, kind, n, dx):
        r = D(0.0)
        ok = self._sbp(kind, n, dx, C.byref(r))
        return bool(ok), r.value

    def mms_bathymetry(self, x, y):
        return self._bath(x, y)

    def mms_state(self, t, x, y):
        o = np.zeros(5)
        self._mstate(t, x, y, _p(o))
        return o

    def mms_state_dt(self, t, x, y):
        o = np.zeros(5)
        self._mstate_dt(t, x, y, _p(o))
        return o

    def mms_source(self, t, x, y, g=9.81):
        o = np.zeros(5)
        self._msrc(t, x, y, g, _p(o))
        return o

    # ref-only ----------------------------------------------------------------
    def run_recorded(self, grid, phys, b, q0, t0, t_final, cfg, out_dir, gauges=(), targets=(), stride=1,
                     source_kind=0):
        """adaptive_solve + RunRecorder + flush() (cli.hpp:100-116): the
        reference writes its CSVs into out_dir.  Returns (q, record)."""
        q0 = np.ascontiguousarray(q0, dtype=np.float64)
        out = np.empty_like(q0)
        rec = Record()
        g = np.ascontiguousarray(np.asarray(gauges, dtype=np.float64).reshape(-1))
        tg = np.ascontiguousarray(np.asarray(targets, dtype=np.float64).reshape(-1))
        self._run_rec(C.byref(grid), C.byref(phys), _p(np.ascontiguousarray(b, np.float64)), source_kind,
                      _p(q0), t0, t_final, C.byref(cfg), _p(out), C.byref(rec), out_dir.encode(),
                      len(g) // 2, _p(g) if len(g) else None, len(tg), _p(tg) if len(tg) else None, int(stride))
        return out, rec

    def prepare(self, name: str, nx=0, ny=0, **params):
        """make_scenario + prepare_run; returns (grid, phys, b, q0, source_kind, t0, t_final)."""
        keys = (C.c_char_p * max(1, len(params)))(*[k.encode() for k in params])
        vals = np.array(list(params.values()) or [0.0], dtype=np.float64)
        g, ph = Grid(), Phys()
        sk, t0, tf = C.c_int(0), D(0.0), D(0.0)
        err = C.create_string_buffer(256)
        st = self._prepare(name.encode(), keys, _p(vals), len(params), nx, ny, C.byref(g), C.byref(ph),
                           None, None, C.byref(sk), C.byref(t0), C.byref(tf), err, 256)
        if st:
            raise ValueError(err.value.decode())
        n = g.nx * g.ny
        b = np.zeros(n)
        q0 = np.zeros(5 * n)
        self._prepare(name.encode(), keys, _p(vals), len(params), g.nx, g.ny, C.byref(g), C.byref(ph),
                      _p(b), _p(q0), C.byref(sk), C.byref(t0), C.byref(tf), err, 256)
        return g, ph, b, q0, sk.value, t0.value, tf.value


# ---------------------------------------------------------------- helpers

def mms_exact_field(grid: Grid, t: float) -> np.ndarray:
    """Manufactured exact state sampled on the grid (numpy restatement of the
    closed form in oracle/hsgn_oracle.c mms_fields; scenarios.hpp:200-214)."""
    nx, ny = grid.nx, grid.ny
    dx = (grid.x_max - grid.x_min) / (nx - 1 if grid.kind_x else nx)
    dy = (grid.y_max - grid.y_min) / (ny - 1 if grid.kind_y else ny)
    x = grid.x_min + np.arange(nx) * dx
    y = grid.y_min + np.arange(ny) * dy
    X, Y = np.meshgrid(x, y)
    tp, fp = 2 * np.pi, 4 * np.pi
    s1x, c1x, s1y, c1y = np.sin(tp * X), np.cos(tp * X), np.sin(tp * Y), np.cos(tp * Y)
    s2x, c2x, s2y, c2y = np.sin(fp * X), np.cos(fp * X), np.sin(fp * Y), np.cos(fp * Y)
    st, ct = np.sin(tp * t), np.cos(tp * t)
    b = (2 / 25) * c1x * c1y + (1 / 25) * c2x * c2y
    bx = -(2 / 25) * tp * s1x * c1y - (1 / 25) * fp * s2x * c2y
    by = -(2 / 25) * tp * c1x * s1y - (1 / 25) * fp * c2x * s2y
    h = 2 + 0.5 * s1x * s1y * ct - b
    u = 0.3 * s1x * st
    v = 0.3 * s1y * st
    ux = 0.3 * tp * c1x * st
    vy = 0.3 * tp * c1y * st
    w = -h * (ux + vy) + 1.5 * (u * bx + v * by)
    return np.concatenate([a.ravel() for a in (h, u, v, w, h)]), b.ravel()


def random_state(n: int, seed: int, lo=0.5, hi=1.5) -> np.ndarray:
    """i.i.d. state in the style of tests/test_rhs.cpp:22-33 (numpy RNG, not
    mt19937: only the distribution matters for these property checks)."""
    rng = np.random.default_rng(seed)
    h = rng.uniform(lo, hi, n)
    u, v, w = rng.uniform(-1, 1, (3, n))
    e = rng.uniform(lo, hi, n)
    return np.concatenate([h, u, v, w, e])


def same_bits(a, b) -> bool:
    """Bit-for-bit equality of two fp64 arrays (distinguishes -0.0 from +0.0
    and compares NaN payloads), stricter than IEEE ==."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
