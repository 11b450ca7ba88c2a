"""Count bit-pattern differences (signed zeros) between the device RHS and the
reference-generated golden outputs (tests/golden/golden_r1.npz)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_02540_b200 as H  # noqa: E402

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden_r1.npz"))
for name in sorted({k.split("/")[1] for k in g.files if k.startswith("rhs/")}):
    a = g[f"rhs/{name}/grid"]
    nx, ny = int(a[0]), int(a[1])
    lam, t, source, variant = g[f"rhs/{name}/par"]
    grid = H.make_grid(a[4], a[5], a[6], a[7], nx, ny, H.BoundaryKind(int(a[2])), H.BoundaryKind(int(a[3])))
    ctx = H.make_rhs_context(grid, H.PhysSetup(9.81, float(lam), 1e-12, g[f"rhs/{name}/b"].reshape(ny, nx)))
    if source:
        ctx.source = "manufactured"
    out = H.StateField(grid)
    (H.rhs_shallow_water if int(variant) == 1 else H.rhs)(ctx, float(t), H.StateField(grid, g[f"rhs/{name}/q"]), out)
    got, want = out.flat(), g[f"rhs/{name}/out"]
    bits = np.count_nonzero(got.view(np.uint64) != want.view(np.uint64))
    print(f"{name:16s} values {got.size:6d}  IEEE != {np.count_nonzero(got != want):5d}  bit patterns differ {bits:5d}"
          f"  zeros in reference {np.count_nonzero(want == 0):5d}")
