"""Pins the CPU oracle against the reference's own known-answer tests
(oracle/kat.cpp ports test_kernel.cpp, test_integrators.cpp, test_quadtree.cpp,
acceptance.cpp criterion 1, ... with the reference's seeds and tolerances)."""
import subprocess


def test_reference_known_answer_tests_pass_on_oracle(oracle):
    res = subprocess.run([oracle.KAT], capture_output=True, text=True)
    print(res.stdout)
    assert res.returncode == 0, res.stdout[-4000:]
    assert "0 failures" in res.stdout
