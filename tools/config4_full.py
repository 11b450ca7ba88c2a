"""BASELINE config 4 at its stated size: 10 fixed BS3 steps of the 8192^2
periodic benchmark workload (manufactured bathymetry and state at t = 0.3,
lambda = 500, dt = 0.25 dx / 20) on the device and with the UNMODIFIED
reference (oracle/_ref, OpenMP on the host cores); full-grid bitwise
comparison of the final states (5 x 67,108,864 values).
Usage: python tools/config4_full.py [steps]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2601_02540_b200 as H  # noqa: E402
from oracle_lib import Oracle, Phys, default_cfg, make_grid as omake  # noqa: E402
from paper_2601_02540_b200.workloads import benchmark_case  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = 8192
g, q, b, lam, dt = benchmark_case(n)
ctx = H.make_rhs_context(g, H.PhysSetup(9.81, lam, 1e-12, b.reshape(n, n)), device=0)
t = time.perf_counter()
dev = H.adaptive_solve(ctx, H.StateField(g, q), 0.0, steps * dt, H.IntegratorConfig(fixed_dt=dt))
t_dev = time.perf_counter() - t
ctx.close()
ref = Oracle("ref")
ref.set_threads(os.cpu_count() or 8)
t = time.perf_counter()
qr, rr = ref.solve(omake(n, n), Phys(9.81, lam, 1e-12), b, q, 0.0, steps * dt, default_cfg(fixed_dt=dt))
t_ref = time.perf_counter() - t
diff = int(np.count_nonzero(dev.q.flat() != qr))
print(f"steps device {dev.accepted} reference {rr.accepted}; t device {dev.t!r} reference {rr.t!r}")
print(f"final state: {diff} of {qr.size} values differ (IEEE ==)")
print(f"wall: device {t_dev:.2f} s (incl. host copies), reference {t_ref:.1f} s on {os.cpu_count()} host threads")
sys.exit(0 if diff == 0 and dev.accepted == rr.accepted and dev.t == rr.t else 1)
