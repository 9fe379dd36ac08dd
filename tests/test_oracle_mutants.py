"""The oracle's pins kill every mutant of tools/mutate_oracle.py (-m "not gpu").

Each mutant writes one plausible mistake into oracle/fdgs_oracle.c (a dropped
term, a wrong sign / index / operand order, a removed clamp) and
runs the pin suites against the mutated build; a surviving mutant would be a
part of the oracle no pin checks.  ~1.5 min on the CPU."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.slow
def test_every_oracle_mutant_is_killed():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "mutate_oracle.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert '"not_killed": []' in r.stdout
