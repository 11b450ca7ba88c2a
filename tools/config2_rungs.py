"""Per-rung cost of the BASELINE config-2 study (manufactured solution,
adaptive BS3 at tol 1e-10, device forcing): wall time, accepted / rejected
attempts and RHS evaluations of each rung.  Usage:
    python tools/config2_rungs.py [t_final] [n1,n2,...] [fixed_dt_cfl]
fixed_dt_cfl > 0: fixed steps dt = cfl * dx instead (the sourced fixed-step path)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200.cli import study_case  # noqa: E402
from paper_2601_02540_b200.scenarios import make_scenario  # noqa: E402

t_final = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
res = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [128, 256, 512, 1024, 2048, 4096]
cfl = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
spec = make_scenario("manufactured")
spec.t_final = t_final
for n in res:
    case = study_case(spec, n, n, 0)
    cfg = H.IntegratorConfig(fixed_dt=cfl * case.grid.dx) if cfl > 0 else H.IntegratorConfig(abs_tol=1e-10, rel_tol=1e-10)
    H.adaptive_solve(case.ctx, case.q0, spec.t0, spec.t0 + 1e-6, cfg)  # warm (graphs, workspaces)
    case.ctx.synchronize()
    t0 = time.perf_counter()
    rec = H.adaptive_solve(case.ctx, case.q0, spec.t0, spec.t_final, cfg)
    case.ctx.synchronize()
    w = time.perf_counter() - t0
    att = rec.accepted + rec.rejected
    print(f"n={n:5d} wall {w:8.3f} s  accepted {rec.accepted:6d} rejected {rec.rejected:5d} rhs {rec.rhs_evals:7d} "
          f"ms/attempt {1e3 * w / max(att, 1):.4f}  t={rec.t:.6f} aborted={rec.aborted}", flush=True)
    rec.device_q.free()
    case.q0.free()
    case.ctx.close()
