"""Fixed-step ms/step of each kernel structure (hsgn_set_fused_stages 0/1/2)
on the benchmark workload, interleaved on one box.  Usage: fusion_ab.py [n] [steps] [reps]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200.workloads import benchmark_case  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g, q, b, lam, dt = benchmark_case(n)
ctx = H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(n, n)), device=0)
y = ctx.state(q)
k1 = ctx.state()
H.rhs(ctx, 0.0, y, k1)
for mode in (0, 1, 2, 3):
    ctx.fused_stages = mode
    H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, steps)  # capture + warm
for rep in range(reps):
    line = []
    for mode in (0, 1, 2, 3):
        ctx.fused_stages = mode
        H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, 4)
        done, ms, kern = H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, steps)
        m = C.c_double(0.0)
        if mode:
            H.api.N.lib().hsgn_profile_fused(ctx._h, y._h, k1._h, dt, 3, C.byref(m))
        line.append(f"mode {mode}: {ms / done:.3f} ms/step ({kern} launches) kernel {m.value:.3f}")
    print(" | ".join(line))
