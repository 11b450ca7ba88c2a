"""GPU test of the NCCL halo-exchange code path on ONE B200.

A 1-rank NCCL communicator attached to a periodic-y context turns it into a
1-slab ring (hsgn_ctx_attach_nccl): ghost-row y edges instead of the index
wrap, direct kernel launches with a grouped ncclSend/ncclRecv after every
kernel, and the halo rows sent to the rank itself.  That is the P-rank
schedule of bench.py --gpus P (slab.make_slab_context) at P = 1, with the
real NCCL calls, so the communicator set-up, the send/recv posting order
(the same-peer case that P = 2 periodic also hits) and the slab kernels run
on hardware.  Required: bitwise equality with the whole-grid context, which
the parity tests pin to the CPU oracle.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200 import slab as S  # noqa: E402
from paper_2601_02540_b200.workloads import mms_fields  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def dist1():
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("nx,ny,kind_x,fused", [(96, 70, 0, 3), (96, 70, 0, 0), (64, 48, 1, 3), (130, 9, 0, 3)])
def test_ring1_matches_whole_grid_bitwise(dist1, nx, ny, kind_x, fused):
    g, q, b = mms_fields(nx, ny, 0.3, kind_x=H.BoundaryKind(kind_x))
    phys = H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(ny, nx))
    dt = 0.25 * g.dx / 20.0
    whole = H.make_rhs_context(g, phys, device=0)
    y1, k1 = whole.state(q), whole.state()
    H.rhs(whole, 0.0, y1, k1)
    k1_host = k1.download().flat().copy()
    H.bs3_fixed_steps(whole, y1, k1, 0.0, dt, 7)
    want_y, want_k = y1.download().flat(), k1.download().flat()

    ring = S.make_slab_context(g, phys, 0, 1, 0, dist1)
    ring.fused_stages = fused
    ry, rk = ring.state(q), ring.state()
    H.rhs(ring, 0.0, ry, rk)
    assert np.count_nonzero(rk.download().flat() != k1_host) == 0
    H.bs3_fixed_steps(ring, ry, rk, 0.0, dt, 7)
    assert np.count_nonzero(ry.download().flat() != want_y) == 0
    assert np.count_nonzero(rk.download().flat() != want_k) == 0
    ring.close()
    whole.close()


def test_ring1_adaptive_matches_whole_grid(dist1):
    nx, ny = 80, 64
    g, q, b = mms_fields(nx, ny, 0.3)
    phys = H.PhysSetup(9.81, 500.0, 1e-12, b.reshape(ny, nx))
    cfg = H.IntegratorConfig(abs_tol=1e-8, rel_tol=1e-8)
    whole = H.make_rhs_context(g, phys, device=0)
    ring = S.make_slab_context(g, phys, 0, 1, 0, dist1)
    a = H.adaptive_solve(whole, H.StateField(g, q), 0.0, 2e-3, cfg)
    r = H.adaptive_solve(ring, H.StateField(g, q), 0.0, 2e-3, cfg)
    assert not a.aborted and not r.aborted
    assert (r.accepted, r.rejected) == (a.accepted, a.rejected)
    assert np.count_nonzero(r.q.flat() != a.q.flat()) == 0
    ring.close()
    whole.close()


@pytest.mark.parametrize("amp,U,dt,floor", [(0.99, 10.0, 1e-3, 1e-12), (0.99, 30.0, 1e-3, 1e-12),
                                             (0.99, 10.0, 1e-3, 0.005)])
@pytest.mark.parametrize("fused", [0, 3])
def test_ring1_failures_match_whole_grid(dist1, amp, U, dt, floor, fused):
    """Depth failures (stage 1, stage 3, floor) on the slab path: the step
    records pass through the cross-rank agreement (hsgn agree_rec) before
    the next kernel and the host read; abort reason, ledger and last valid
    state equal the whole-grid run's (which test_gpu_fused pins to the
    reference)."""
    nx, ny = 64, 48
    x = -1 + np.arange(nx) * 2 / nx
    y = -1 + np.arange(ny) * 2 / ny
    X, Y = np.meshgrid(x, y)
    e = np.exp(-(X ** 2 + Y ** 2) / 0.05)
    h = 1 - amp * e
    q = np.concatenate([h.ravel(), (U * X * e).ravel(), (U * Y * e).ravel(), np.zeros(nx * ny), h.ravel()])
    g = H.make_grid(-1.0, 1.0, -1.0, 1.0, nx, ny)
    phys = H.PhysSetup(9.81, 500.0, 1e-12, np.zeros((ny, nx)))
    cfg = H.IntegratorConfig(fixed_dt=dt, h_floor=floor)
    whole = H.make_rhs_context(g, phys, device=0)
    whole.fused_stages = fused
    ring = S.make_slab_context(g, phys, 0, 1, 0, dist1)
    ring.fused_stages = fused
    a = H.adaptive_solve(whole, H.StateField(g, q), 0.0, 200 * dt, cfg)
    r = H.adaptive_solve(ring, H.StateField(g, q), 0.0, 200 * dt, cfg)
    assert a.aborted and r.aborted
    assert r.abort_reason == a.abort_reason
    assert (r.accepted, r.rejected, r.rhs_evals, r.t) == (a.accepted, a.rejected, a.rhs_evals, a.t)
    assert np.count_nonzero(r.q.flat() != a.q.flat()) == 0
    ring.close()
    whole.close()
