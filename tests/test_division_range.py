"""CPU: the fast correctly rounded division of the stage kernels
(sgn_device.cuh div_fast) in the deep-subnormal regime that its high-word
range test lets through (tools/div_hole_check.c, seeded, 2e7 quotients with
a zero high word): bit-identical to IEEE a / h."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_deep_subnormal_quotients_match_ieee_division(tmp_path):
    exe = str(tmp_path / "div_hole_check")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", os.path.join(ROOT, "tools", "div_hole_check.c"), "-o", exe,
                    "-lm"], check=True)
    r = subprocess.run([exe, "20000000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0
    tested, bad = (int(w) for w in r.stdout.split()[1::2])
    assert tested > 1000000 and bad == 0, r.stdout
