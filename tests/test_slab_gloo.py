"""Multi-rank slab decomposition on CPU (gloo, world_size 2 and 3).

The library's multi-GPU path (hsgn_ctx_create_slab + NCCL halo exchange,
hsgn_host.cu exchange()) cuts the grid into y-slabs with ghost rows above
and below and exchanges the rows just written after every kernel: per stage
(k2, ynew, k4; one row needed) or, with the default fused structure, ynew
after S12 and k4 after S3 (two rows).  These tests run both schedules with
torch.distributed/gloo as the transport and
the CPU oracle as the stage arithmetic, and require the gathered P-rank
state to be BIT-IDENTICAL to the single-domain reference solve (the RHS has
no reductions, so decomposition must not change a single bit).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_02540_b200 import slab as S


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_and_neighbours():
    assert S.partition(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert S.partition(8192, 8)[-1] == (7168, 8192)
    with pytest.raises(ValueError):
        S.partition(5, 3)
    assert S.neighbours(0, 4, True) == (3, 1)
    assert S.neighbours(3, 4, True) == (2, 0)
    assert S.neighbours(0, 4, False) == (-1, 1)
    assert S.neighbours(3, 4, False) == (2, -1)


def _exchange_fn(rank, nranks, periodic_y):
    dn, up = S.neighbours(rank, nranks, periodic_y)

    def exchange(send_dn, send_up):
        # two phases (downward, then upward) so that every (src, dst) pair
        # carries one message per phase: no reliance on tag matching
        r_dn = r_up = None
        reqs = []
        if dn >= 0:
            reqs.append(dist.isend(torch.from_numpy(send_dn), dn))
        if up >= 0:
            r_up = torch.empty(send_up.shape[0], dtype=torch.float64)
            reqs.append(dist.irecv(r_up, up))
        for r in reqs:
            r.wait()
        reqs = []
        if up >= 0:
            reqs.append(dist.isend(torch.from_numpy(send_up), up))
        if dn >= 0:
            r_dn = torch.empty(send_dn.shape[0], dtype=torch.float64)
            reqs.append(dist.irecv(r_dn, dn))
        for r in reqs:
            r.wait()
        return (r_dn.numpy() if r_dn is not None else None, r_up.numpy() if r_up is not None else None)

    return exchange


def _worker(rank, nranks, port, kind_y, steps, q_shared, result, schedule="stage"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from oracle_lib import Oracle, Phys, make_grid as omake

        orc = Oracle("orc")
        orc.set_threads(1)
        nx, ny = 32, 24
        periodic = kind_y == 0
        g = omake(nx, ny, kind_x=0, kind_y=kind_y)
        dx = 2.0 / nx
        dy = 2.0 / (ny - 1 if kind_y else ny)
        q0 = np.frombuffer(q_shared[0], dtype=np.float64).reshape(5, ny, nx)
        b = np.frombuffer(q_shared[1], dtype=np.float64).reshape(ny, nx)
        j0, j1 = S.partition(ny, nranks)[rank]
        n_loc = j1 - j0
        dn, up = S.neighbours(rank, nranks, periodic)
        exch = _exchange_fn(rank, nranks, periodic)
        ph = Phys(9.81, 500.0, 1e-12)

        def ghosted(field):  # (5, n_loc, nx) -> (5, n_loc + 2, nx) via the halo exchange
            return np.stack([S.ghost_rows(field[f], rank, nranks, periodic, exch) for f in range(5)])

        bg = S.ghost_rows(b[j0:j1], rank, nranks, periodic, exch)
        # local evaluation grid: the ghost-extended slab; a wall-side slab keeps
        # the wall closure at its true face (ghost rows are discarded)
        lg = omake(nx, n_loc + 2, kind_x=0, kind_y=1 if (kind_y and (dn < 0 or up < 0)) else 0)
        lo = 1 if dn >= 0 else 0  # where the slab's row 0 sits in the extended array
        if dn < 0:  # bottom wall: extended array = slab rows + ghost above (+1 pad row)
            pass

        def rhs_slab(qext):
            """Tendency of the slab rows from a ghost-extended stage input."""
            if dn >= 0 and up >= 0:
                arr, bb = qext, bg
            elif dn < 0:  # drop the (zero) ghost row below: wall face is local row 0
                arr, bb = qext[:, 1:], bg[1:]
            else:  # drop the ghost row above: wall face is the local last row
                arr, bb = qext[:, :-1], bg[:-1]
            rows = arr.shape[1]
            gg = omake(nx, rows, kind_x=0, kind_y=lg.kind_y)
            out = np.empty(5 * rows * nx)
            st = orc._lib_rhs_dxdy(gg, dx, dy, ph, np.ascontiguousarray(bb).ravel(), np.ascontiguousarray(arr).ravel(),
                                   out)
            assert st == 0
            out = out.reshape(5, rows, nx)
            if dn >= 0 and up >= 0:
                return out[:, 1:-1]
            if dn < 0:
                return out[:, :-1]
            return out[:, 1:]

        y = q0[:, j0:j1].copy()
        dt = 0.25 * dx / 20.0
        k1 = rhs_slab(ghosted(y))

        # ---- the default fixed-step structure S12 + S3:
        # two ghost rows per side, halos of ynew after S12 and of k4 after S3
        lo2, hi2 = (2 if dn >= 0 else 0), (2 if up >= 0 else 0)
        wall_kind = 1 if (kind_y and (dn < 0 or up < 0)) else 0

        def ext2(field):  # (n_loc, nx) -> two exchanged ghost rows on each interior side
            fb, fa = exch(field[:2].ravel().copy() if dn >= 0 else None,
                          field[-2:].ravel().copy() if up >= 0 else None)
            parts = ([fb.reshape(2, nx)] if dn >= 0 else []) + [field] + ([fa.reshape(2, nx)] if up >= 0 else [])
            return np.concatenate(parts, axis=0)

        def ext2_state(qs):
            return np.stack([ext2(qs[f]) for f in range(5)])

        def rhs_rows(arr, bb):  # tendencies of every row of an extended array (edges invalid)
            rows = arr.shape[1]
            gg = omake(nx, rows, kind_x=0, kind_y=wall_kind)
            out = np.empty(5 * rows * nx)
            assert orc._lib_rhs_dxdy(gg, dx, dy, ph, np.ascontiguousarray(bb).ravel(),
                                     np.ascontiguousarray(arr).ravel(), out) == 0
            return out.reshape(5, rows, nx)

        b2 = ext2(b[j0:j1])
        if schedule == "s12":
            y_e, k1_e = ext2_state(y), ext2_state(k1)
            for _ in range(steps):
                k2_e = rhs_rows(y_e + (0.5 * dt) * k1_e, b2)           # S12: stage 1 on slab rows -1..n
                s0, s1 = (1 if dn >= 0 else 0), y_e.shape[1] - (1 if up >= 0 else 0)
                q2 = (y_e + (0.75 * dt) * k2_e)[:, s0:s1]              # stage-2 input, rows -1..n
                k3 = rhs_rows(q2, b2[s0:s1])[:, lo2 - s0:lo2 - s0 + n_loc]
                yy, kk1, kk2 = y_e[:, lo2:lo2 + n_loc], k1_e[:, lo2:lo2 + n_loc], k2_e[:, lo2:lo2 + n_loc]
                ynew = yy + (dt * (2.0 / 9.0)) * kk1 + (dt * (1.0 / 3.0)) * kk2 + (dt * (4.0 / 9.0)) * k3
                y_e = ext2_state(ynew)                                  # ynew halo (2 rows)
                k4 = rhs_rows(y_e, b2)[:, lo2:lo2 + n_loc]              # S3
                k1_e = ext2_state(k4)                                   # k4 halo (2 rows)
            y = y_e[:, lo2:lo2 + n_loc]
            steps_left = 0
        elif schedule == "overlap":
            # the overlapped slab schedule of hsgn_host.cu enqueue_slab_step:
            # S12 on the two-row edge bands -> ynew halo exchange -> S12 on the
            # interior band -> S3 on the edge bands -> k4 halo exchange -> S3 on
            # the interior band.  Every band is evaluated from ONLY the rows it
            # reads (2 beyond it for S12, 1 for S3), so the exchanges provably
            # need nothing but the edge bands.
            G = 2

            def band(fn, reach, j_a, j_b, *arrs):
                """Rows [j_a, j_b) of fn(sub-arrays of the extended arrays
                holding slab rows [j_a - reach, j_b + reach), clipped at a wall)."""
                a = max(lo2 + j_a - reach, 0)
                e = min(lo2 + j_b + reach, arrs[0].shape[1])
                out = fn(*[x[:, a:e] if x.ndim == 3 else x[a:e] for x in arrs])
                return out[:, lo2 + j_a - a:lo2 + j_b - a]

            def s12(ys, ks, bs):
                k2 = rhs_rows(ys + (0.5 * dt) * ks, bs)
                k3 = rhs_rows(ys + (0.75 * dt) * k2, bs)
                return ys + (dt * (2.0 / 9.0)) * ks + (dt * (1.0 / 3.0)) * k2 + (dt * (4.0 / 9.0)) * k3

            def s3(ys, bs):
                return rhs_rows(ys, bs)

            def exch_rows(lo_rows, hi_rows, interior):
                """Assemble the slab from its bands and add the exchanged
                ghost rows (two per interior side), as the comm stream does."""
                full = np.concatenate([lo_rows, interior, hi_rows], axis=1)
                return np.stack([ext2(full[f]) for f in range(5)])

            y_e, k1_e = ext2_state(y), ext2_state(k1)
            for _ in range(steps):
                yn_lo = band(s12, 2, 0, G, y_e, k1_e, b2)
                yn_hi = band(s12, 2, n_loc - G, n_loc, y_e, k1_e, b2)
                # (the exchange below only reads yn_lo / yn_hi)
                yn_in = band(s12, 2, G, n_loc - G, y_e, k1_e, b2)
                yn_e = exch_rows(yn_lo, yn_hi, yn_in)
                k4_lo = band(s3, 1, 0, G, yn_e, b2)
                k4_hi = band(s3, 1, n_loc - G, n_loc, yn_e, b2)
                k4_in = band(s3, 1, G, n_loc - G, yn_e, b2)
                y_e, k1_e = yn_e, exch_rows(k4_lo, k4_hi, k4_in)
            y = y_e[:, lo2:lo2 + n_loc]
            steps_left = 0
        else:
            steps_left = steps
        for _ in range(steps_left):
            yg, k1g = ghosted(y), ghosted(k1)
            k2 = rhs_slab(yg + (0.5 * dt) * k1g)                    # stage 1 (then k2 halo)
            k2g = ghosted(k2)
            k3 = rhs_slab(yg + (0.75 * dt) * k2g)                   # stage 2
            ynew = y + (dt * (2.0 / 9.0)) * k1 + (dt * (1.0 / 3.0)) * k2 + (dt * (4.0 / 9.0)) * k3
            k4 = rhs_slab(ghosted(ynew))                            # stage 3 (ynew halo before it)
            y, k1 = ynew, k4                                        # FSAL swap
        # gather on rank 0
        t = torch.from_numpy(np.ascontiguousarray(y).ravel())
        sizes = [(b1 - b0) for b0, b1 in S.partition(ny, nranks)]
        if rank == 0:
            parts = [torch.empty(5 * s * nx, dtype=torch.float64) for s in sizes]
            parts[0] = t
            for r in range(1, nranks):
                dist.recv(parts[r], r)
            full = np.concatenate([p.numpy().reshape(5, s, nx) for p, s in zip(parts, sizes)], axis=1)
            result.put(full.ravel().tobytes())
        else:
            dist.send(t, 0)
    finally:
        dist.destroy_process_group()


def _oracle_lib_patch():
    # orc_rhs_dxdy binding (added here to keep oracle_lib's generic loader small)
    import ctypes as C

    from oracle_lib import PD, Grid, Oracle, Phys

    def rhs_dxdy(self, grid, dx, dy, phys, b, q, out):
        fn = self.lib.orc_rhs_dxdy
        fn.restype = C.c_int
        fn.argtypes = [C.POINTER(Grid), C.c_double, C.c_double, C.POINTER(Phys), PD, C.c_int, C.c_double, PD, PD]
        return fn(C.byref(grid), dx, dy, C.byref(phys), b.ctypes.data_as(PD), 0, 0.0, q.ctypes.data_as(PD),
                  out.ctypes.data_as(PD))

    Oracle._lib_rhs_dxdy = rhs_dxdy


@pytest.mark.parametrize("schedule", ["stage", "s12", "overlap"])
@pytest.mark.parametrize("nranks,kind_y", [(2, 0), (3, 0), (2, 1), (3, 1)])
def test_slab_bs3_bitwise_equals_single_domain(nranks, kind_y, schedule):
    """schedule "stage": one ghost row, halos after every stage (the
    per-stage kernels); "s12": two ghost rows, halos of ynew after S12 and
    of k4 after S3 (the default fused structure); "overlap": the same with
    edge-band / interior-band launches, the exchanges reading only the edge
    bands (the NCCL slab schedule, hsgn_host.cu enqueue_slab_step)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracle_lib import Oracle, Phys, default_cfg, make_grid as omake, mms_exact_field
    _oracle_lib_patch()
    nx, ny, steps = 32, 24, 5
    g = omake(nx, ny, kind_x=0, kind_y=kind_y)
    q0, b = mms_exact_field(g, 0.3)
    dt = 0.25 * (2.0 / nx) / 20.0
    # single-domain reference: the plain BS3 stage sequence (no end clipping),
    # itself pinned to the reference's adaptive_solve(fixed_dt) in test_oracle
    orc = Oracle("orc")
    want = q0.copy()
    k1 = np.zeros_like(q0)
    import ctypes as C
    from oracle_lib import PD
    assert orc._fixed(C.byref(g), C.byref(Phys(9.81, 500.0, 1e-12)), b.ctypes.data_as(PD), want.ctypes.data_as(PD),
                      k1.ctypes.data_as(PD), 0.0, dt, steps, 1) == 0

    class rec:  # noqa: N801
        accepted = steps
    ctx = mp.get_context("spawn")
    q_shared = (ctx.RawArray("b", q0.tobytes()), ctx.RawArray("b", b.tobytes()))
    result = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker_entry,
                         args=(r, nranks, port, kind_y, rec.accepted, q_shared, result, schedule))
             for r in range(nranks)]
    for p in procs:
        p.start()
    got = np.frombuffer(result.get(timeout=240), dtype=np.float64)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got, want), np.count_nonzero(got != want)


def _worker_entry(*args):
    _oracle_lib_patch()
    _worker(*args)
