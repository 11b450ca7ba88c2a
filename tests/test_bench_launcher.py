"""bench.py's multi-GPU bookkeeping on CPU (no GPU needed).

* ``--gpus N`` outside torchrun launches N ranks itself, and refuses (exit 2,
  a JSON line with ``error``) when fewer than N GPUs are visible instead of
  timing fewer GPUs than it reports;
* with gloo and world_size 2 / 3, every rank's share of the weak- and
  strong-scaling workloads (periodic config-4 input and the reflecting
  gaussian_obstacle basin) tiles the global grid and equals the rows of the
  single-process sample bit for bit, and the max-over-ranks timing
  reduction takes the slowest rank.
"""
import json
import os
import socket
import subprocess
import sys
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _visible_gpus():
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30).stdout
        return sum(1 for line in out.splitlines() if line.startswith("GPU "))
    except Exception:
        return 0


@pytest.mark.parametrize("inside_torchrun", [False, True])
def test_gpus_beyond_visible_refused(inside_torchrun):
    n = max(2, _visible_gpus() + 1)
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    if inside_torchrun:  # a rank of an N-rank launch on a node with fewer GPUs
        env.update(WORLD_SIZE=str(n), RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "2"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == n and "error" in line
    assert "refusing" in r.stderr


def _args(**kw):
    a = dict(scaling="weak", config5=False, n=0, rows=0, ny=0, bc="periodic", gpus=1)
    a.update(kw)
    return SimpleNamespace(**a)


def test_shapes():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.shapes(_args(), 1) == (8192, 8192, "weak")           # config 4
    assert bench.shapes(_args(), 8) == (8192, 65536, "weak")          # 8192-row slabs
    assert bench.shapes(_args(config5=True), 4) == (16384, 16384, "weak")  # 16384 x 4096 per GPU
    assert bench.shapes(_args(scaling="strong"), 2) == (16384, 16384, "strong")
    assert bench.shapes(_args(scaling="strong", config5=True, n=32768), 8) == (32768, 32768, "strong")


def _worker(rank, world, port, cases, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        import bench
        from paper_2601_02540_b200 import slab as S
        from paper_2601_02540_b200.workloads import bench_case
        res = []
        for kw in cases:
            nx, ny, _ = bench.shapes(_args(**kw), world)
            j0, j1 = S.partition(ny, world)[rank]
            g, q, b, lam, dt, aux = bench_case(kw["bc"], nx, ny, rows=(j0, j1))
            rows = torch.tensor([j0, j1], dtype=torch.int64)
            allr = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(allr, rows)
            n_loc = (j1 - j0) * nx
            width = 6 * max(int(r[1] - r[0]) for r in allr) * nx  # gloo all_gather: equal sizes
            mine = np.zeros(width)
            mine[:6 * n_loc] = np.concatenate([q, b])
            parts = [torch.zeros(width, dtype=torch.float64) for _ in allr]
            dist.all_gather(parts, torch.from_numpy(mine))
            t = torch.tensor([float(rank + 1)], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)   # bench.py max_over_ranks
            res.append(([tuple(r.tolist()) for r in allr], [p.numpy() for p in parts], float(t.item()), lam, dt,
                        n_loc))
        if rank == 0:
            out.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_shares_tile_the_global_workload(world):
    sys.path.insert(0, ROOT)
    import bench
    from paper_2601_02540_b200.workloads import bench_case
    cases = [dict(bc="periodic", n=64, rows=18), dict(bc="reflecting", n=64, rows=18),
             dict(bc="periodic", n=64, ny=60, scaling="strong"), dict(bc="reflecting", n=48, ny=50, scaling="strong")]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = out.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for kw, (rows, parts, tmax, lam, dt, _) in zip(cases, res):
        nx, ny, _ = bench.shapes(_args(**kw), world)
        assert rows[0][0] == 0 and rows[-1][1] == ny
        assert all(rows[k][1] == rows[k + 1][0] for k in range(world - 1))
        g, q, b, lam1, dt1, _ = bench_case(kw["bc"], nx, ny)
        assert (lam, dt) == (lam1, dt1)
        q = q.reshape(5, ny, nx)
        b = b.reshape(ny, nx)
        for (j0, j1), part in zip(rows, parts):
            m = (j1 - j0) * nx
            assert np.array_equal(part[:5 * m].reshape(5, j1 - j0, nx), q[:, j0:j1])
            assert np.array_equal(part[5 * m:6 * m].reshape(j1 - j0, nx), b[j0:j1])
        assert tmax == float(world)
