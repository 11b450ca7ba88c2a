"""Diagnose device-vs-reference differences on the reflecting basin (config 3
at 512^2): first differing step, locations, and which kernel structure /
tile split produces them.  GPU only; run under gpurun."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2601_02540_b200 as H  # noqa: E402
from oracle_lib import Oracle, default_cfg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ref = Oracle("ref")
ref.set_threads(os.cpu_count() or 8)
orc = Oracle("orc")
g, ph, b, q0, sk, t0, tf = ref.prepare("gaussian_obstacle", n, n, bounded=1.0)
grid = H.make_grid(g.x_min, g.x_max, g.y_min, g.y_max, g.nx, g.ny, g.kind_x, g.kind_y)
dt = 0.25 * min(grid.dx, grid.dy) / 20.0


def where(a, b):
    d = np.nonzero(a != b)[0]
    out = []
    for k in d[:20]:
        f, r = divmod(int(k), n * n)
        j, i = divmod(r, n)
        out.append((f, i, j, a[k], b[k]))
    return len(d), out


# RHS on q0
ctx = H.make_rhs_context(grid, H.PhysSetup(ph.g, ph.lambda_, ph.h_floor, b.reshape(n, n)))
print("stencil kind", ctx.stencil_kind)
qt = H.StateField(grid)
H.rhs(ctx, 0.0, H.StateField(grid, q0), qt)
st, want, _ = ref.rhs(g, ph, b, q0)
print("rhs(q0) vs ref:", where(qt.flat(), want))
st, want2, _ = orc.rhs(g, ph, b, q0)
print("orc rhs(q0) vs ref:", where(want2, want))

for steps in (1, 2, 4, 8, 16, 32, 64, 128, 200):
    want, rr = ref.solve(g, ph, b, q0, t0, t0 + steps * dt, default_cfg(fixed_dt=dt))
    wo, ro = orc.solve(g, ph, b, q0, t0, t0 + steps * dt, default_cfg(fixed_dt=dt))
    line = [f"steps={steps} ref acc={rr.accepted}", f"orc-vs-ref {where(wo, want)[0]}"]
    for mode in (0, 3):
        for rpb in (0, 7, 1000):
            c2 = H.make_rhs_context(grid, H.PhysSetup(ph.g, ph.lambda_, ph.h_floor, b.reshape(n, n)))
            c2.fused_stages = mode
            if rpb:
                c2.set_rows_per_block(rpb)
            dev = H.adaptive_solve(c2, H.StateField(grid, q0), t0, t0 + steps * dt, H.IntegratorConfig(fixed_dt=dt))
            nd, locs = where(dev.q.flat(), want)
            line.append(f"m{mode}/rpb{rpb}:{nd}")
            if nd and steps <= 8:
                print(f"  mode {mode} rpb {rpb} steps {steps}: first diffs {locs[:8]}")
            c2.close()
    print(" ".join(line), flush=True)
