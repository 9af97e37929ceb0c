"""The CPU oracle against the reference's own known-answer tests.

tests/oracle_kat.cpp ports /root/reference/proj/tests/*.cpp and acceptance
criteria 1, 2, 4, 7 case by case (same seeds, inputs and tolerances); the
oracle must pass all of them before any GPU result is compared with it.
"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_oracle_known_answers():
    exe = os.path.join(ROOT, "oracle", "build", "oracle_kat")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:]
    assert "0 failures" in r.stdout
    # every ported reference case ran
    assert r.stdout.count("[PASS]") >= 60
