"""On-device run recorder: the reference's RunRecorder (io.hpp:107-219) and its
CSV writers (io.hpp:19-59), backed by hsgn_recorder_* (include/hsgn_b200.h).

The reference samples gauges, computes three serial full-grid reductions
every `conservation_stride` accepted steps and copies the whole state after
every step (for the closer-neighbour snapshot rule).  Here the device does
the sampling inside the fixed-step CUDA graphs, one fused row-sum pass per
conservation row, and snapshots are stream-ordered copies of whichever of the
integrator's two state buffers holds the chosen state -- no per-step state
copy and no host round trip between records.

Usage mirrors cli.hpp:100-116:

    rec = RunRecorder(ctx, out_dir, gauges, snapshot_times, stride)
    sol = adaptive_solve(ctx, q0, t0, t_final, cfg, recorder=rec)
    rec.flush()            # gauges.csv, conservation.csv (+ snapshot CSVs)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np

from . import _native as N


def fmt17(v: float) -> str:
    """io.hpp:19-23: %.17g (round-trip exact)."""
    return "%.17g" % v


def fmt_short(v: float) -> str:
    """io.hpp:26-30: %g for file names."""
    return "%g" % v


@dataclass
class GaugeNode:
    """io.hpp:32-35"""
    i: int
    j: int
    x: float
    y: float


@dataclass
class SnapshotRecord:
    """io.hpp:96-100"""
    target: float
    actual: float
    path: str


@dataclass
class ConsRow:
    t: float
    mass: float
    energy: float
    energy_rate: float


def _grid_xy(grid) -> Tuple[np.ndarray, np.ndarray]:
    i = np.arange(grid.nx, dtype=np.float64)
    j = np.arange(grid.ny, dtype=np.float64)
    return grid.x_min + i * grid.dx, grid.y_min + j * grid.dy  # Grid2D::x / y (grid.hpp:24-25)


def _rows_csv(path: str, header: str, cols: Sequence[np.ndarray]) -> None:
    data = np.column_stack([np.asarray(c, dtype=np.float64) for c in cols])
    with open(path, "w") as f:
        f.write(header)
        np.savetxt(f, data, fmt="%.17g", delimiter=",")


def write_snapshot_csv(path: str, grid, q: np.ndarray, b: np.ndarray) -> None:
    """io.hpp:50-59: x,y,h,u,v,w,eta,b per node, x fastest, %.17g."""
    n = grid.nx * grid.ny
    q = np.asarray(q, dtype=np.float64).reshape(5, n)
    x, y = _grid_xy(grid)
    X = np.tile(x, grid.ny)
    Y = np.repeat(y, grid.nx)
    _rows_csv(path, "x,y,h,u,v,w,eta,b\n", [X, Y, *q, np.asarray(b, np.float64).reshape(n)])


def write_cross_section_csv(path: str, grid, q: np.ndarray, b: np.ndarray, y_target: float) -> None:
    """io.hpp:62-77: the grid row nearest to y_target."""
    node = nearest_node(grid, grid.x_min, y_target)
    q = np.asarray(q, dtype=np.float64).reshape(5, grid.ny, grid.nx)[:, node.j]
    x, _ = _grid_xy(grid)
    bj = np.asarray(b, np.float64).reshape(grid.ny, grid.nx)[node.j]
    _rows_csv(path, "# cross section along y = " + fmt17(node.y) + "\nx,h,u,v,w,eta,b\n", [x, *q, bj])


def nearest_node(grid, x: float, y: float) -> GaugeNode:
    """io.hpp:38-48 (std::lround rounds halves away from zero)."""
    def lround(v):
        return int(np.floor(v + 0.5)) if v >= 0 else -int(np.floor(-v + 0.5))
    i = min(max(lround((x - grid.x_min) / grid.dx), 0), grid.nx - 1)
    j = min(max(lround((y - grid.y_min) / grid.dy), 0), grid.ny - 1)
    return GaugeNode(i, j, grid.x_min + i * grid.dx, grid.y_min + j * grid.dy)


class RunRecorder:
    """io.hpp:107-219 on the device.  Attach with adaptive_solve(...,
    recorder=rec); snapshot CSVs are written when the solve returns (the
    reference writes them as the target is crossed), gauges.csv and
    conservation.csv by flush()."""

    def __init__(self, ctx, out_dir: str, gauge_positions: Sequence[Sequence[float]] = (),
                 snapshot_targets: Sequence[float] = (), conservation_stride: int = 1):
        self.ctx = ctx
        self.dir = out_dir
        g = np.ascontiguousarray(np.asarray(gauge_positions, dtype=np.float64).reshape(-1))
        tg = np.ascontiguousarray(np.asarray(snapshot_targets, dtype=np.float64).reshape(-1))
        self._h = C.c_void_p()
        st = N.lib().hsgn_recorder_create(ctx._h, len(g) // 2, g.ctypes.data_as(N.PD) if len(g) else None,
                                          len(tg), tg.ctypes.data_as(N.PD) if len(tg) else None,
                                          int(conservation_stride), C.byref(self._h))
        if st:
            msg = N.lib().hsgn_last_error(ctx._h).decode()
            from .api import HsgnError
            raise (ValueError if st == N.HSGN_EINVAL else HsgnError)(f"RunRecorder: {msg}")
        self._snaps: List[SnapshotRecord] = []

    # ---------------------------------------------------------------- queries
    def _counts(self):
        g, c, s = C.c_int64(0), C.c_int64(0), C.c_int32(0)
        N.lib().hsgn_recorder_counts(self._h, C.byref(g), C.byref(c), C.byref(s))
        return g.value, c.value, s.value

    def gauge_nodes(self) -> List[GaugeNode]:
        out, k = [], 0
        i, j, x, y = C.c_int32(), C.c_int32(), C.c_double(), C.c_double()
        while N.lib().hsgn_recorder_gauge_node(self._h, k, C.byref(i), C.byref(j), C.byref(x), C.byref(y)) == 0:
            out.append(GaugeNode(i.value, j.value, x.value, y.value))
            k += 1
        return out

    def gauge_series(self) -> Tuple[np.ndarray, np.ndarray]:
        """(t[rows], values[rows, n_gauges]) of h + b at the gauge nodes."""
        rows = self._counts()[0]
        ng = len(self.gauge_nodes())
        t = np.zeros(rows)
        v = np.zeros(rows * ng)
        N.lib().hsgn_recorder_gauges(self._h, t.ctypes.data_as(N.PD), v.ctypes.data_as(N.PD))
        return t, v.reshape(rows, ng)

    def conservation_rows(self) -> List[ConsRow]:
        rows = self._counts()[1]
        a = np.zeros(4 * rows)
        if rows:
            N.lib().hsgn_recorder_conservation(self._h, a.ctypes.data_as(N.PD))
        return [ConsRow(*a[4 * k:4 * k + 4]) for k in range(rows)]

    def snapshot_state(self, k: int) -> Tuple[float, float, np.ndarray]:
        grid = self.ctx.grid
        q = np.zeros(5 * grid.nx * grid.ny)
        tg, ac = C.c_double(), C.c_double()
        st = N.lib().hsgn_recorder_snapshot(self._h, k, C.byref(tg), C.byref(ac), q.ctypes.data_as(N.PD))
        if st:
            raise IndexError(k)
        return tg.value, ac.value, q

    def snapshots(self) -> List[SnapshotRecord]:
        self.write_snapshots()
        return list(self._snaps)

    # ---------------------------------------------------------------- output
    def write_snapshots(self) -> None:
        """take_snapshot (io.hpp:197-204) for every snapshot not yet on disk."""
        n = self._counts()[2]
        while len(self._snaps) < n:
            k = len(self._snaps)
            target, actual, q = self.snapshot_state(k)
            path = self.dir + "/snapshot_t" + fmt_short(target) + ".csv"
            os.makedirs(self.dir, exist_ok=True)
            write_snapshot_csv(path, self.ctx.grid, q, self.ctx.bathymetry())
            self._snaps.append(SnapshotRecord(target, actual, path))

    def flush(self) -> None:
        """io.hpp:155-185: gauges.csv (if any gauge) and conservation.csv."""
        os.makedirs(self.dir, exist_ok=True)
        self.write_snapshots()
        nodes = self.gauge_nodes()
        if nodes:
            t, v = self.gauge_series()
            head = "".join(f"# gauge_{k + 1} at ({fmt17(g.x)}, {fmt17(g.y)})\n" for k, g in enumerate(nodes))
            head += "t" + "".join(f",gauge_{k + 1}" for k in range(len(nodes))) + "\n"
            _rows_csv(self.dir + "/gauges.csv", head, [t, *v.T])
        rows = self.conservation_rows()
        _rows_csv(self.dir + "/conservation.csv", "t,total_mass,total_energy,semidiscrete_energy_rate\n",
                  [[r.t for r in rows], [r.mass for r in rows], [r.energy for r in rows],
                   [r.energy_rate for r in rows]])

    def close(self) -> None:
        if self._h:
            N.lib().hsgn_recorder_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
