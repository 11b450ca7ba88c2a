"""BASELINE config 1 at its stated size and length: the solitary wave
(soliton_1d defaults, lambda = 30000, periodic [-30, 30]^2) on a 256 x 256
grid, fixed-step BS3 (dt = 1.5e-3) for one full traversal
t = 60 / C (~11,660 steps), on the device and with the UNMODIFIED reference
(oracle/_ref, OpenMP on the host cores) from the reference's own initial
state.  Reports bitwise equality of the final states and the L2 errors
against the exact translated profile.  Usage: python tools/config1_full.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2601_02540_b200 as H  # noqa: E402
from oracle_lib import Oracle, default_cfg  # noqa: E402
from paper_2601_02540_b200.scenarios import exact_state, make_scenario, prepare_run  # noqa: E402

ref = Oracle("ref")
ref.set_threads(os.cpu_count() or 8)
g, ph, b, q0, sk, t0, tf = ref.prepare("soliton", 256, 256)
dt = 1.5e-3
spec = make_scenario("soliton")
run = prepare_run(spec, 256, 256, device=0)
assert np.count_nonzero(run.q0.download().flat() != q0) == 0, "initial states differ"
t = time.perf_counter()
dev = H.adaptive_solve(run.ctx, run.q0, t0, tf, H.IntegratorConfig(fixed_dt=dt))
t_dev = time.perf_counter() - t
t = time.perf_counter()
qr, rr = ref.solve(g, ph, b, q0, t0, tf, default_cfg(fixed_dt=dt))
t_ref = time.perf_counter() - t
diff = int(np.count_nonzero(dev.q.flat() != qr))
ex = exact_state(spec, 256, 256, dev.t)
n = 256 * 256
errs = {v: float(H.discrete_l2_error(run.ctx, dev.device_q, H.StateField(run.grid, ex), f)) for f, v in
        ((0, "h"), (1, "u"))}
print(f"steps device {dev.accepted} reference {rr.accepted}; t device {dev.t!r} reference {rr.t!r}")
print(f"final state: {diff} of {5 * n} values differ (IEEE ==)")
print(f"L2 error vs exact at t = {dev.t:.6g}: {errs}")
print(f"wall: device {t_dev:.2f} s, reference {t_ref:.1f} s on {os.cpu_count()} host threads")
sys.exit(0 if diff == 0 and dev.accepted == rr.accepted and dev.t == rr.t else 1)
