"""Slab domain decomposition over the GPUs of one box.

The grid is cut into y-slabs of contiguous rows (x fastest, so the halo
rows are one contiguous span per field).  Each rank keeps two ghost rows
above and below its slab (the fused stage-1+2 kernel reads two rows beyond
the rows it finishes); after every kernel the library exchanges the freshly
written boundary rows with the two neighbours (ring wrap when y is
periodic) through NCCL send/recv on its own stream.  Because ghost values
are formed by the same expressions as interior ones, the P-rank state is
bitwise equal to the 1-rank state (the RHS has no reductions).  The
host-side reference below exchanges one row (what a single stage needs).

torch.distributed is the plumbing only: it carries the ncclUniqueId from
rank 0 to the others and provides barriers / the max-over-ranks timing.
The partition arithmetic below is shared with the CPU (gloo) tests.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Tuple

import numpy as np


def partition(ny: int, nranks: int) -> List[Tuple[int, int]]:
    """Contiguous near-equal row ranges [j0, j1) per rank (first ranks take
    the remainder); every slab has at least 2 rows."""
    if nranks < 1 or ny < 2 * nranks:
        raise ValueError(f"cannot cut {ny} rows into {nranks} slabs of >= 2 rows")
    base, rem = divmod(ny, nranks)
    out, j = [], 0
    for r in range(nranks):
        k = base + (1 if r < rem else 0)
        out.append((j, j + k))
        j += k
    return out


def neighbours(rank: int, nranks: int, periodic_y: bool) -> Tuple[int, int]:
    """(below, above) neighbour ranks; -1 where a wall closes the domain."""
    dn = rank - 1 if rank > 0 else (nranks - 1 if periodic_y else -1)
    up = rank + 1 if rank + 1 < nranks else (0 if periodic_y else -1)
    return dn, up


def ghost_rows(field: np.ndarray, rank: int, nranks: int, periodic_y: bool, exchange) -> np.ndarray:
    """Reference implementation of one halo exchange on host arrays:
    returns the slab extended by its two ghost rows (zeros at walls).
    `exchange(send_below, send_above) -> (from_below, from_above)` is the
    transport (torch.distributed gloo in tests, NCCL in the library)."""
    dn, up = neighbours(rank, nranks, periodic_y)
    from_below, from_above = exchange(field[0].copy() if dn >= 0 else None,
                                      field[-1].copy() if up >= 0 else None)
    lo = from_below if from_below is not None else np.zeros_like(field[0])
    hi = from_above if from_above is not None else np.zeros_like(field[0])
    return np.concatenate([lo[None], field, hi[None]], axis=0)


def slab_fields(nx: int, ny: int, t: float, rank: int, nranks: int):
    """The benchmark workload restricted to this rank's rows."""
    from .workloads import mms_fields
    j0, j1 = partition(ny, nranks)[rank]
    return mms_fields(nx, ny, t, rows=(j0, j1))  # only this rank's rows are sampled


class SlabGroup:
    """In-process slab decomposition (hsgn_group_*): n slabs on `devices`
    (default: all on the current device), halo rows pulled over (peer)
    device pointers after every stage.  Host arrays are the full grid."""

    def __init__(self, grid, phys, n: int, devices=None):
        from . import _native as N
        self.N = N
        self.grid, self.n = grid, n
        b = np.ascontiguousarray(phys.b if phys.b is not None else np.zeros((grid.ny, grid.nx)), dtype=np.float64)
        g = grid.c_struct()
        ph = N.hsgn_phys(phys.g, phys.lambda_, phys.h_floor)
        devs = (C.c_int * n)(*(devices or [-1] * n))
        self._h = C.c_void_p()
        st = N.lib().hsgn_group_create(C.byref(g), C.byref(ph), b.ctypes.data_as(N.PD), devs, n, C.byref(self._h))
        if st:
            raise RuntimeError(f"hsgn_group_create failed ({st})")
        self.rows = partition(grid.ny, n)

    def _check(self, st, what):
        if st:
            msg = self.N.lib().hsgn_group_last_error(self._h)
            raise RuntimeError(f"{what}: status {st} {msg.decode() if msg else ''}")

    def state(self, host=None):
        s = C.c_void_p()
        self._check(self.N.lib().hsgn_group_state_alloc(self._h, C.byref(s)), "state_alloc")
        if host is not None:
            self.upload(s, host)
        return s

    def upload(self, s, host):
        a = np.ascontiguousarray(host, dtype=np.float64).reshape(-1)
        self._check(self.N.lib().hsgn_group_state_upload(self._h, s, a.ctypes.data_as(self.N.PD)), "upload")

    def download(self, s):
        out = np.empty(5 * self.grid.nx * self.grid.ny)
        self._check(self.N.lib().hsgn_group_state_download(self._h, s, out.ctypes.data_as(self.N.PD)), "download")
        return out

    def rhs(self, t, q, out):
        bad = C.c_int64(0)
        self._check(self.N.lib().hsgn_group_rhs(self._h, float(t), q, out, C.byref(bad)), "rhs")

    def bs3_fixed_steps(self, y, k1, t, dt, steps):
        done = C.c_int64(0)
        self._check(self.N.lib().hsgn_group_bs3_fixed_steps(self._h, y, k1, float(t), float(dt), int(steps),
                                                             C.byref(done)), "bs3_fixed_steps")
        return done.value

    def reduce(self, kind, q, qt=None):
        out = C.c_double(0.0)
        self._check(self.N.lib().hsgn_group_reduce(self._h, int(kind), q, qt, C.byref(out)), "reduce")
        return out.value

    def close(self):
        if self._h:
            self.N.lib().hsgn_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_slab_context(grid, phys, rank: int, nranks: int, device: int, dist):
    """Create this rank's slab context and attach an NCCL communicator whose
    unique id is broadcast from rank 0 over torch.distributed."""
    import torch

    from . import _native as N
    from .api import RhsContext
    j0, j1 = partition(grid.ny, nranks)[rank]
    ctx = RhsContext(grid, phys, device=device, slab=(j0, j1, rank, nranks))
    uid = (C.c_char * 128)()
    if rank == 0:
        st = N.lib().hsgn_nccl_unique_id(uid)
        if st != 0:
            raise RuntimeError("hsgn_nccl_unique_id failed")
    t = torch.tensor(list(bytes(uid)) if rank == 0 else [0] * 128, dtype=torch.uint8, device=f"cuda:{device}")
    dist.broadcast(t, src=0)
    raw = bytes(t.cpu().tolist())
    st = N.lib().hsgn_ctx_attach_nccl(ctx._h, raw)
    if st != 0:
        raise RuntimeError("hsgn_ctx_attach_nccl: " + N.lib().hsgn_last_error(ctx._h).decode())
    return ctx
