"""BASELINE config 2 at its stated sizes: the manufactured-solution refinement
study with variable bathymetry, periodic, 128^2 .. 4096^2 on one B200,
through the CLI's convergence driver (cli.run_convergence_study, adaptive
BS3 at the reference's study tolerance 1e-10, device forcing terms).
Prints the reference-format convergence table.  Usage:
    python tools/config2_ladder.py [t_final] [out_dir]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_02540_b200 as H  # noqa: E402
from paper_2601_02540_b200 import cli  # noqa: E402
from paper_2601_02540_b200.scenarios import make_scenario  # noqa: E402

t_final = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/config2_ladder"
os.makedirs(out, exist_ok=True)
spec = make_scenario("manufactured")
spec.t_final = t_final
res = [128, 256, 512, 1024, 2048, 4096]
t0 = time.perf_counter()
table = cli.run_convergence_study(spec, res, H.IntegratorConfig(abs_tol=1e-10, rel_tol=1e-10))
wall = time.perf_counter() - t0
cli.write_convergence_csv(os.path.join(out, "convergence.csv"), table)
print(open(os.path.join(out, "convergence.csv")).read())
print(f"t_final {t_final}  wall {wall:.1f} s")
