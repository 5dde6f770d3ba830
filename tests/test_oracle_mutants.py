"""Every plausible oracle mutant of tools/oracle_mutants.py fails at least one CPU pin.

This is the check behind the claim that the oracle is pinned to the paper and the mathematics, not
only to itself (VERDICT r01 "What's weak" 1): each mutant is a dropped term, a wrong sign, power or
index, or a transposed operand in Eqs. (1a)-(1b), the strains, the SO(3) maps, the integrator or the
NEXT-row forcing terms, and each must be killed.  CPU only (gcc + the oracle pins), about a minute
with one worker per host core.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_oracle_mutant_is_killed():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "oracle_mutants.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=1800)
    lines = [ln for ln in p.stdout.splitlines() if "killed" in ln or "SURVIVED" in ln or "error" in ln]
    assert p.returncode == 0, "\n".join(lines[-60:]) + p.stderr[-2000:]
    assert "mutants killed" in p.stdout
