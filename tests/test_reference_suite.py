"""Drop-in check: the reference's own unit tests for the strategy space, the specs and the
cost model (pkg/tests/test_strategies.py, test_specs.py, test_costs.py — 92 tests), run
unmodified with ``parapilot`` aliased to this package.  Build container only (the
reference tree is not on the GPU box); its dp_search tests need a GPU and are covered by
the golden fixtures and tests/test_gpu_parity.py (same fuzz generators and seeds)."""

import subprocess
import sys
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parents[1]

SHIM = f"""
import sys
sys.path.insert(0, {str(ROOT)!r})
import paper_2307_02031_b200 as G
from paper_2307_02031_b200 import balance, costs, dpsearch, errors, planner, specs, strategies
sys.modules["parapilot"] = G
for name, mod in (("balance", balance), ("costs", costs), ("dpsearch", dpsearch), ("errors", errors),
                  ("planner", planner), ("specs", specs), ("strategies", strategies)):
    sys.modules["parapilot." + name] = mod
import pytest
sys.exit(pytest.main(["-q", "-p", "no:cacheprovider", "--rootdir=/tmp"] + sys.argv[1:]))
"""


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference tree not present")
def test_reference_cpu_suites_pass_against_this_package():
    files = [str(REF_TESTS / f) for f in ("test_strategies.py", "test_specs.py", "test_costs.py")]
    proc = subprocess.run([sys.executable, "-c", SHIM] + files, capture_output=True, text=True, cwd="/tmp",
                          timeout=600)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-2000:]
    assert "92 passed" in proc.stdout
