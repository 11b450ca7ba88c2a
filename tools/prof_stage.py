"""Small driver for ncu / A-B timing: one RHS + `steps` fused BS3 steps at n x n.
Usage: python tools/prof_stage.py [n] [steps] [rows_per_block] [x] [bc]
  bc: periodic (config 4 workload, default) | walls (the same manufactured
  state on the bounded grid [-1,1]^2: closures + SAT, stencil kind 0)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200.workloads import benchmark_case, mms_fields  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rpb = int(sys.argv[3]) if len(sys.argv) > 3 else 0
bc = sys.argv[5] if len(sys.argv) > 5 else "periodic"
if bc == "walls":
    B = H.BoundaryKind.bounded
    g, q, b = mms_fields(n, n, 0.3, kind_x=B, kind_y=B)
    lam, dt = 500.0, 0.25 * g.dx / 20.0
else:
    g, q, b, lam, dt = benchmark_case(n)
ctx = H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(n, n)), device=0)
if rpb:
    ctx.set_rows_per_block(rpb)
y = ctx.state(q)
k1 = ctx.state()
H.rhs(ctx, 0.0, y, k1)
done, ms, kern = H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, steps)
print(f"n={n} bc={bc} kind={ctx.stencil_kind} steps={done} ms/step={ms / max(done, 1):.3f} kernels={kern} "
      f"(first call, incl. capture)")
if len(sys.argv) > 4 and sys.argv[4] != "-":
    import ctypes as C
    H.set_kernel_timing(ctx, True)
    for rep in range(3):
        H.prepare_fixed_steps(ctx, y, k1, dt, steps)
        done, ms, kern = H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, steps)
        s12, s3, nt = H.kernel_times(ctx)
        ms3 = (C.c_double * 3)()
        H.api.N.lib().hsgn_profile_stages(ctx._h, y._h, k1._h, dt, 3, ms3)
        print(f"rep {rep}: ms/step={ms / max(done, 1):.3f} in-graph S12={s12:.3f} S3={s3:.3f} ({nt} steps) "
              f"per-stage S1,S2,S3={[round(x, 3) for x in ms3]}")
