import ctypes as C, sys, os, time, subprocess, threading
sys.path.insert(0, os.getcwd())
import paper_2601_02540_b200 as H
from paper_2601_02540_b200.workloads import benchmark_case
n = 8192
g, q, b, lam, dt = benchmark_case(n)
ctx = H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(n, n)), device=0)
y = ctx.state(q); k1 = ctx.state(); H.rhs(ctx, 0.0, y, k1)
L = H.api.N.lib()
def prof(reps):
    m = C.c_double(0); L.hsgn_profile_fused(ctx._h, y._h, k1._h, dt, reps, C.byref(m))
    s = (C.c_double*3)(); L.hsgn_profile_stages(ctx._h, y._h, k1._h, dt, reps, s)
    return m.value, s[2]
def clocks():
    out = subprocess.run(["nvidia-smi","--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active","--format=csv,noheader"],capture_output=True,text=True).stdout.strip()
    return out
for steps in (50, 300):
    H.prepare_fixed_steps(ctx, y, k1, dt, steps); H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, 4)
    res = []
    def samp():
        for _ in range(6): res.append(clocks()); time.sleep(0.1)
    th = threading.Thread(target=samp); th.start()
    done, ms, kern = H.bs3_fixed_steps(ctx, y, k1, 0.0, dt, steps)
    th.join()
    print("steps", steps, "ms/step", ms/done, res[:4])
for reps in (3, 60):
    print("reps", reps, "S12, S3 ms", prof(reps))
