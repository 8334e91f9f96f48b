"""The C++ drop-in (paper_2603_10242_b200/dropin/prover_b200.cpp) in place of
the reference's proj/src/prover.cpp: the reference's OWN acceptance gate
(proj/tests/acceptance.cpp, all ten criteria — including wire exactness,
forgery resistance, O(1) verification at N = 100,000, and the simulator's
finality timelines and determinism, all of which call prove_block /
verify_finality_certificate) relinked against it, run on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2603_10242_b200", "lib", "ace_acceptance_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in not built (needs /root/reference)")
def test_reference_acceptance_gate_with_gpu_prover():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "acceptance: all criteria passed" in r.stdout
    for crit in (1, 6, 8):
        assert f"criterion {crit:2d} [PASS]" in r.stdout
