"""Host-side mirror of the reference's operator API for the hot path.

Same names, argument meaning and error behaviour as the reference C++
library (/root/reference/proj/include/hsgn), backed by the sm_100a kernels
through the C ABI (include/hsgn_b200.h):

    reference (file:line)                        here
    -------------------------------------------  -------------------------------
    BoundaryKind           grid.hpp:11           BoundaryKind
    Grid2D / make_grid     grid.hpp:16-68        Grid2D / make_grid
    StateField             model.hpp:22-35       StateField (host, numpy)
    PhysSetup              model.hpp:40-45       PhysSetup
    depth_error            model.hpp:15-17       DepthError
    RhsContext / make_rhs_context  rhs.hpp:17-54 RhsContext / make_rhs_context
    rhs / rhs_periodic / rhs_reflecting / rhs_shallow_water  rhs.hpp:219-248
    init_auxiliary         model.hpp:93-105      init_auxiliary
    total_mass / total_energy  model.hpp:77-87   total_mass / total_energy
    energy_rate            analysis.hpp:47-67    energy_rate
    discrete_l2_error      analysis.hpp:15-25    discrete_l2_error
    IntegratorConfig / SolutionRecord / adaptive_solve  time_integration.hpp:18-350

States may be host ``StateField`` objects (copied in/out around each call)
or device-resident ``DeviceState`` handles (no copies).  Nothing here
computes on the CPU: every operator launches the native kernels, and the
native library must be loadable (no fallback).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Union

import numpy as np

from . import _native as N


class DepthError(RuntimeError):
    """hsgn::depth_error (model.hpp:15-17): non-positive depth somewhere."""


class HsgnError(RuntimeError):
    pass


class BoundaryKind(enum.IntEnum):
    periodic = 0
    bounded = 1


@dataclass
class Grid2D:
    """grid.hpp:16-41.  Periodic spacing excludes the seam (L/n); bounded
    includes both endpoints (L/(n-1))."""
    x_min: float = 0.0
    x_max: float = 1.0
    y_min: float = 0.0
    y_max: float = 1.0
    nx: int = 0
    ny: int = 0
    dx: float = 0.0
    dy: float = 0.0
    kind_x: BoundaryKind = BoundaryKind.periodic
    kind_y: BoundaryKind = BoundaryKind.periodic

    def x(self, i):
        return self.x_min + np.asarray(i) * self.dx

    def y(self, j):
        return self.y_min + np.asarray(j) * self.dy

    def n_total(self) -> int:
        return self.nx * self.ny

    def sample(self, f) -> np.ndarray:
        """Field (ny, nx) with f(x_i, y_j) at every node (grid.hpp:56-63)."""
        X, Y = np.meshgrid(self.x(np.arange(self.nx)), self.y(np.arange(self.ny)))
        return np.ascontiguousarray(np.broadcast_to(f(X, Y), (self.ny, self.nx)), dtype=np.float64)

    def c_struct(self) -> N.hsgn_grid:
        return N.hsgn_grid(self.nx, self.ny, int(self.kind_x), int(self.kind_y),
                           self.x_min, self.x_max, self.y_min, self.y_max)


def direction_spacing(lo: float, hi: float, n: int, kind: BoundaryKind) -> float:
    return (hi - lo) / n if kind == BoundaryKind.periodic else (hi - lo) / (n - 1)


def make_grid(x_min, x_max, y_min, y_max, nx, ny, kind_x=BoundaryKind.periodic,
              kind_y=BoundaryKind.periodic) -> Grid2D:
    """grid.hpp:47-68, same validation and messages."""
    if not (x_max > x_min) or not (y_max > y_min):
        raise ValueError("make_grid: domain extents must be increasing")
    if nx < 4 or ny < 4:
        raise ValueError(f"make_grid: need at least 4 nodes per direction, got nx={nx} ny={ny}")
    kx, ky = BoundaryKind(kind_x), BoundaryKind(kind_y)
    return Grid2D(float(x_min), float(x_max), float(y_min), float(y_max), int(nx), int(ny),
                  direction_spacing(x_min, x_max, nx, kx), direction_spacing(y_min, y_max, ny, ky), kx, ky)


class StateField:
    """Host state h, u, v, w, eta; storage is one (5, ny, nx) fp64 array so a
    state is the 5 contiguous fields of the C ABI host layout."""
    names = ("h", "u", "v", "w", "eta")
    n_fields = 5

    def __init__(self, grid_or_shape, data: Optional[np.ndarray] = None):
        if isinstance(grid_or_shape, Grid2D):
            shape = (grid_or_shape.ny, grid_or_shape.nx)
        else:
            shape = tuple(grid_or_shape)
        if data is None:
            self.data = np.zeros((5,) + shape, dtype=np.float64)
        else:
            self.data = np.ascontiguousarray(np.asarray(data, dtype=np.float64).reshape((5,) + shape))

    h = property(lambda s: s.data[0])
    u = property(lambda s: s.data[1])
    v = property(lambda s: s.data[2])
    w = property(lambda s: s.data[3])
    eta = property(lambda s: s.data[4])

    def fields(self):
        return [self.data[k] for k in range(5)]

    def copy(self) -> "StateField":
        return StateField(self.data.shape[1:], self.data.copy())

    def flat(self) -> np.ndarray:
        return self.data.reshape(-1)


@dataclass
class PhysSetup:
    """model.hpp:40-45"""
    g: float = 9.81
    lambda_: float = 500.0
    h_floor: float = 1e-12
    b: Optional[np.ndarray] = None


def _check(ctx: Optional["RhsContext"], st: int, what: str):
    if st == N.HSGN_OK:
        return
    msg = N.lib().hsgn_last_error(ctx._h if ctx is not None else None)
    msg = msg.decode() if msg else ""
    if st == N.HSGN_EDEPTH:
        raise DepthError(msg)
    if st == N.HSGN_EINVAL:
        raise ValueError(f"{what}: invalid argument {msg}")
    raise HsgnError(f"{what}: {N.STATUS_NAMES.get(st, st)} {msg}")


class DeviceState:
    """Device-resident StateField (opaque hsgn_state)."""

    def __init__(self, ctx: "RhsContext", host: Optional[Union[StateField, np.ndarray]] = None):
        self.ctx = ctx
        self._h = N.STATE()
        _check(ctx, N.lib().hsgn_state_alloc(ctx._h, C.byref(self._h)), "hsgn_state_alloc")
        if host is not None:
            self.upload(host)

    @classmethod
    def borrow(cls, ctx, handle) -> "DeviceState":
        s = cls.__new__(cls)
        s.ctx = ctx
        s._h = N.STATE(handle)
        s._borrowed = True
        return s

    def upload(self, host):
        arr = host.flat() if isinstance(host, StateField) else np.ascontiguousarray(host, np.float64).reshape(-1)
        assert arr.size == 5 * self.ctx.ny_local * self.ctx.grid.nx
        _check(self.ctx, N.lib().hsgn_state_upload(self.ctx._h, self._h, arr.ctypes.data_as(N.PD)),
               "hsgn_state_upload")

    def download(self, out: Optional[StateField] = None) -> StateField:
        out = out if out is not None else StateField((self.ctx.ny_local, self.ctx.grid.nx))
        _check(self.ctx, N.lib().hsgn_state_download(self.ctx._h, self._h, out.data.ctypes.data_as(N.PD)),
               "hsgn_state_download")
        return out

    def copy_from(self, other: "DeviceState"):
        _check(self.ctx, N.lib().hsgn_state_copy(self.ctx._h, other._h, self._h), "hsgn_state_copy")

    def field_ptr(self, f: int) -> int:
        p = N.PD()
        _check(self.ctx, N.lib().hsgn_state_field_ptr(self._h, f, C.byref(p)), "hsgn_state_field_ptr")
        return C.cast(p, C.c_void_p).value

    def free(self):
        if getattr(self, "_borrowed", False):
            return
        if self._h and self.ctx._h:
            N.lib().hsgn_state_free(self.ctx._h, self._h)
        self._h = N.STATE()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class RhsContext:
    """rhs.hpp:17-38: grid, physics, SBP operators, bathymetry, workspace and
    the optional source hook, living on one B200."""

    def __init__(self, grid: Grid2D, phys: PhysSetup, device: int = -1, slab=None):
        b = phys.b if phys.b is not None else np.zeros((grid.ny, grid.nx))
        b = np.ascontiguousarray(b, dtype=np.float64)
        self.grid, self.phys = grid, phys
        self._h = N.CTX()
        g = grid.c_struct()
        ph = N.hsgn_phys(phys.g, phys.lambda_, phys.h_floor)
        L = N.lib()
        if slab is None:
            if b.size != grid.nx * grid.ny:
                raise ValueError("make_rhs_context: bathymetry shape must match grid")
            st = L.hsgn_ctx_create(C.byref(g), C.byref(ph), b.ctypes.data_as(N.PD), device, C.byref(self._h))
            self.j_begin, self.j_end, self.rank, self.nranks = 0, grid.ny, 0, 1
        else:
            j0, j1, rank, nranks = slab
            if b.size != grid.nx * (j1 - j0):
                raise ValueError("slab bathymetry must hold the slab rows")
            st = L.hsgn_ctx_create_slab(C.byref(g), C.byref(ph), b.ctypes.data_as(N.PD), device, j0, j1,
                                        rank, nranks, C.byref(self._h))
            self.j_begin, self.j_end, self.rank, self.nranks = j0, j1, rank, nranks
        if st != N.HSGN_OK:
            if st == N.HSGN_EINVAL:
                raise ValueError("make_rhs_context: invalid grid/physics")
            raise HsgnError(f"hsgn_ctx_create failed: {N.STATUS_NAMES.get(st, st)} (is a B200 visible?)")
        self.ny_local = self.j_end - self.j_begin
        self._source = None
        self._b = b

    def bathymetry(self) -> np.ndarray:
        """ctx.phys.b of this context's rows (host copy)."""
        return self._b

    # ctx.source (rhs.hpp:24-26): None or "manufactured"
    @property
    def source(self):
        return self._source

    @source.setter
    def source(self, kind):
        k = {None: 0, "manufactured": 1}[kind]
        _check(self, N.lib().hsgn_set_source(self._h, k), "hsgn_set_source")
        self._source = kind

    @property
    def n_evals(self) -> int:
        return int(N.lib().hsgn_n_evals(self._h))

    def set_rows_per_block(self, rows: int):
        _check(self, N.lib().hsgn_set_rows_per_block(self._h, rows), "hsgn_set_rows_per_block")

    @property
    def stencil_kind(self) -> int:
        """0 general, 1 power-of-two, 2 common-factor (all bit-identical)."""
        return int(N.lib().hsgn_stencil_kind(self._h))

    @stencil_kind.setter
    def stencil_kind(self, kind: int):
        _check(self, N.lib().hsgn_set_stencil_kind(self._h, int(kind)), "hsgn_set_stencil_kind")

    @property
    def fused_stages(self) -> int:
        """Fixed-step / attempt kernel structure: 0 one kernel per stage,
        3 (default) stages 1 + 2 fused (S12), then stage 3."""
        return int(N.lib().hsgn_fused_stages(self._h))

    @fused_stages.setter
    def fused_stages(self, mode):
        _check(self, N.lib().hsgn_set_fused_stages(self._h, int(mode)), "set_fused_stages")

    def state(self, host=None) -> DeviceState:
        return DeviceState(self, host)

    def synchronize(self):
        _check(self, N.lib().hsgn_synchronize(self._h), "hsgn_synchronize")

    def close(self):
        if self._h:
            N.lib().hsgn_ctx_destroy(self._h)
            self._h = N.CTX()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_rhs_context(grid: Grid2D, phys: PhysSetup, device: int = -1) -> RhsContext:
    return RhsContext(grid, phys, device)


# ----------------------------------------------------------------- operators

def _as_device(ctx, q):
    if isinstance(q, DeviceState):
        return q, False
    return DeviceState(ctx, q), True


def _rhs_common(ctx: RhsContext, t: float, q, out, shallow: bool):
    dq, _ = _as_device(ctx, q)
    dout = out if isinstance(out, DeviceState) else DeviceState(ctx)
    bad = C.c_int64(0)
    fn = N.lib().hsgn_rhs_shallow_water if shallow else N.lib().hsgn_rhs
    _check(ctx, fn(ctx._h, float(t), dq._h, dout._h, C.byref(bad)), "rhs")
    if not isinstance(out, DeviceState):
        dout.download(out)
    return out


def rhs(ctx: RhsContext, t: float, q, out):
    """rhs.hpp:236-238; raises DepthError (out untouched) on !(h > 0)."""
    return _rhs_common(ctx, t, q, out, False)


def rhs_periodic(ctx: RhsContext, t: float, q, out):
    assert ctx.grid.kind_x == BoundaryKind.periodic and ctx.grid.kind_y == BoundaryKind.periodic
    return _rhs_common(ctx, t, q, out, False)


def rhs_reflecting(ctx: RhsContext, t: float, q, out):
    assert ctx.grid.kind_x == BoundaryKind.bounded or ctx.grid.kind_y == BoundaryKind.bounded
    return _rhs_common(ctx, t, q, out, False)


def rhs_shallow_water(ctx: RhsContext, t: float, q, out):
    return _rhs_common(ctx, t, q, out, True)


def init_auxiliary(ctx: RhsContext, q):
    """model.hpp:93-105 (in place): eta = h, w from the SBP operators."""
    dq, tmp = _as_device(ctx, q)
    _check(ctx, N.lib().hsgn_init_auxiliary(ctx._h, dq._h), "init_auxiliary")
    if tmp:
        dq.download(q)
    return q


def _reduce(ctx, fn, *states):
    ds = [_as_device(ctx, s)[0] for s in states]
    out = C.c_double(0.0)
    _check(ctx, fn(ctx._h, *[d._h for d in ds], C.byref(out)), fn.__name__)
    return out.value


def total_mass(ctx: RhsContext, q) -> float:
    return _reduce(ctx, N.lib().hsgn_total_mass, q)


def total_energy(ctx: RhsContext, q) -> float:
    return _reduce(ctx, N.lib().hsgn_total_energy, q)


def energy_rate(ctx: RhsContext, q, q_t) -> float:
    return _reduce(ctx, N.lib().hsgn_energy_rate, q, q_t)


def mass_weighted_sum(ctx: RhsContext, q, field_index: int) -> float:
    """sbp.hpp:219-239 of one field of a state (SBP-norm quadrature)."""
    dq = _as_device(ctx, q)[0]
    out = C.c_double(0.0)
    _check(ctx, N.lib().hsgn_mass_weighted_sum(ctx._h, dq._h, field_index, C.byref(out)), "mass_weighted_sum")
    return out.value


def discrete_l2_error(ctx: RhsContext, a, b, field_index: int) -> float:
    da, db = _as_device(ctx, a)[0], _as_device(ctx, b)[0]
    out = C.c_double(0.0)
    _check(ctx, N.lib().hsgn_discrete_l2_error(ctx._h, da._h, db._h, field_index, C.byref(out)),
           "discrete_l2_error")
    return out.value


def eoc(err_coarse: float, err_fine: float, dx_coarse: float, dx_fine: float) -> float:
    """analysis.hpp:29-39 (host arithmetic, not on the hot path)."""
    if not (dx_coarse > 0.0) or not (dx_fine > 0.0) or dx_coarse == dx_fine:
        raise ValueError("eoc: spacings must be positive and distinct")
    if err_coarse < 0.0 or err_fine < 0.0:
        raise ValueError("eoc: errors must be non-negative")
    if err_fine == 0.0:
        return math.inf
    if err_coarse == 0.0:
        return -math.inf
    return math.log(err_coarse / err_fine) / math.log(dx_coarse / dx_fine)


# ----------------------------------------------------------------- integrator

@dataclass
class IntegratorConfig:
    """time_integration.hpp:18-29"""
    abs_tol: float = 1e-6
    rel_tol: float = 1e-6
    dt_initial: float = 0.0
    dt_max: float = math.inf
    safety: float = 0.9
    growth_cap: float = 5.0
    shrink_floor: float = 0.2
    max_steps: int = 50_000_000
    fixed_dt: float = 0.0
    h_floor: float = 1e-12

    def c_struct(self) -> N.hsgn_cfg:
        return N.hsgn_cfg(self.abs_tol, self.rel_tol, self.dt_initial, self.dt_max, self.safety,
                          self.growth_cap, self.shrink_floor, int(self.max_steps), self.fixed_dt, self.h_floor)


@dataclass
class SolutionRecord:
    """time_integration.hpp:33-42"""
    q: Optional[StateField] = None
    t: float = 0.0
    accepted: int = 0
    rejected: int = 0
    rhs_evals: int = 0
    rhs_evals_setup: int = 0
    aborted: bool = False
    abort_reason: str = ""


AcceptObserver = Callable[[float, DeviceState, DeviceState], None]


def adaptive_solve(ctx: RhsContext, q0, t0: float, t_final: float, cfg: IntegratorConfig = None,
                   on_accept: Optional[AcceptObserver] = None, out: Optional[DeviceState] = None,
                   recorder=None) -> SolutionRecord:
    """time_integration.hpp:209-350 on the fused device pipeline.  The RHS is
    the context's own split form (the generic callable of the reference
    cannot be fused into stage kernels).  on_accept receives device states
    valid only during the call; ``recorder`` (a recorder.RunRecorder) is the
    on-device AcceptObserver of cli.hpp:100-111."""
    cfg = cfg or IntegratorConfig()
    dq0, _ = _as_device(ctx, q0)
    dout = out if out is not None else DeviceState(ctx)
    rec = N.hsgn_record()
    cfgc = cfg.c_struct()
    err_box = []

    def _obs(t, qh, qth, user):
        try:
            on_accept(t, DeviceState.borrow(ctx, qh), DeviceState.borrow(ctx, qth))
        except BaseException as e:  # surface after the native call returns
            err_box.append(e)

    cb = N.OBSERVER(_obs) if on_accept is not None else N.OBSERVER()
    st = N.lib().hsgn_solve_recorded(ctx._h, dq0._h, float(t0), float(t_final), C.byref(cfgc), dout._h,
                                     C.byref(rec), cb, None, recorder._h if recorder is not None else None)
    if err_box:
        raise err_box[0]
    _check(ctx, st, "adaptive_solve")
    if recorder is not None:
        recorder.write_snapshots()
    res = SolutionRecord(None, rec.t, rec.accepted, rec.rejected, rec.rhs_evals, rec.rhs_evals_setup,
                         bool(rec.aborted), rec.reason.decode())
    res.q = dout.download() if out is None else None
    res.device_q = dout
    return res


def prepare_fixed_steps(ctx: RhsContext, y: DeviceState, k1: DeviceState, dt: float, steps: int) -> None:
    """Build the CUDA graphs bs3_fixed_steps(ctx, y, k1, ..., dt, steps) will
    launch (one-time host work; no step is run)."""
    _check(ctx, N.lib().hsgn_prepare_fixed_steps(ctx._h, y._h, k1._h, float(dt), int(steps)),
           "prepare_fixed_steps")


def set_kernel_timing(ctx: RhsContext, on: bool) -> None:
    """Event nodes around every kernel of the fixed-step graphs (whole grid,
    S12 + S3): kernel_times() then gives the per-kernel durations measured
    inside the last bs3_fixed_steps call."""
    _check(ctx, N.lib().hsgn_set_kernel_timing(ctx._h, int(bool(on))), "set_kernel_timing")


def kernel_times(ctx: RhsContext):
    """(mean S12 ms, mean S3 ms, steps timed) of the last bs3_fixed_steps."""
    a, b, n = C.c_double(0.0), C.c_double(0.0), C.c_int64(0)
    _check(ctx, N.lib().hsgn_kernel_times(ctx._h, C.byref(a), C.byref(b), C.byref(n)), "kernel_times")
    return a.value, b.value, n.value


def bs3_fixed_steps(ctx: RhsContext, y: DeviceState, k1: DeviceState, t: float, dt: float, steps: int):
    """The bare fused fixed-step pipeline (benchmark entry): returns
    (steps_done, device_ms, kernels)."""
    done = C.c_int64(0)
    _check(ctx, N.lib().hsgn_bs3_fixed_steps(ctx._h, y._h, k1._h, float(t), float(dt), int(steps),
                                             C.byref(done)), "bs3_fixed_steps")
    ms = C.c_double(0.0)
    kern = C.c_int64(0)
    N.lib().hsgn_last_timing(ctx._h, C.byref(ms), C.byref(kern))
    return done.value, ms.value, kern.value
