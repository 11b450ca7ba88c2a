import os, sys
sys.path.insert(0, os.getcwd())
import paper_2601_02540_b200 as H
from paper_2601_02540_b200.workloads import benchmark_case
n = 8192
g, q, b, lam, dt = benchmark_case(n)
ctx = H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(n, n)), device=0)
ctx.fused_stages = 2
y = ctx.state(q); k1 = ctx.state(); H.rhs(ctx, 0.0, y, k1)
print(H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, 4))
