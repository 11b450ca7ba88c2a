"""ms per adaptive attempt (per-stage vs S12 + S3) on the benchmark workload.
Usage: adaptive_ab.py [n] [t_final_in_dt]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200.workloads import benchmark_case  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
m = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g, q, b, lam, dt = benchmark_case(n)
ctx = H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(n, n)), device=0)
y = ctx.state(q)
out = ctx.state()
for rep in range(2):
    for mode in (0, 3):
        ctx.fused_stages = mode
        t0 = time.perf_counter()
        r = H.adaptive_solve(ctx, y, 0.0, m * dt, H.IntegratorConfig(abs_tol=1e-6, rel_tol=1e-6, dt_initial=dt, dt_max=dt), out=out)
        el = time.perf_counter() - t0
        att = r.accepted + r.rejected
        print(f"mode {mode}: {att} attempts, {1e3 * el / att:.3f} ms/attempt (wall, incl. the initial RHS)")
