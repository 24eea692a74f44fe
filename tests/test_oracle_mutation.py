"""The oracle's choice pins are not vacuous: tests/mutation_check.sh rebuilds the oracle with
one-token mutations of the Eq. 3 argmin (ties, direction, strict descent) and of the Eq. 4
argmin (ties, direction, locks) and requires tests/test_oracle_choice.py to fail against each
mutant.  -m "not gpu" (gcc + the CPU pins, ~1 min)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_choice_mutant_is_killed():
    r = subprocess.run(["bash", os.path.join(ROOT, "tests", "mutation_check.sh")], capture_output=True,
                       text=True, timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("killed:") == 8
