"""Small driver for ncu: one RHS + `steps` fused BS3 steps on the benchmark
workload (config 4) at n x n.  Usage: python tools/prof_stage.py [n] [steps] [rows_per_block]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200.workloads import benchmark_case  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rpb = int(sys.argv[3]) if len(sys.argv) > 3 else 0
g, q, b, lam, dt = benchmark_case(n)
ctx = H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(n, n)), device=0)
if rpb:
    ctx.set_rows_per_block(rpb)
y = ctx.state(q)
k1 = ctx.state()
H.rhs(ctx, 0.0, y, k1)
done, ms, kern = H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, steps)
print(f"n={n} steps={done} ms/step={ms / max(done, 1):.3f} kernels={kern} (first call, incl. capture)")
if len(sys.argv) > 4:
    import ctypes as C
    for rep in range(3):
        done, ms, kern = H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, steps)
        ms3 = (C.c_double * 3)()
        H.api.N.lib().hsgn_profile_stages(ctx._h, y._h, k1._h, dt, 3, ms3)
        m31 = C.c_double(0.0)
        H.api.N.lib().hsgn_profile_fused(ctx._h, y._h, k1._h, dt, 3, C.byref(m31))
        print(f"rep {rep}: ms/step={ms / max(done, 1):.3f} stages={[round(x, 3) for x in ms3]} "
              f"S31={m31.value:.3f}")
