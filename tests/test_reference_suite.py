"""Drop-in check: the reference's own unit tests for the hot-path modules,
compiled unchanged (oracle/Makefile) once against the reference library and
once against include/elaskit + libelaskit_b200.so, must produce identical
per-assertion outcomes — including the reference's known defects
(test_migration.cpp:107 and :147/:150), which the B200 build
reproduces because parity follows the implementation, not the assertions."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "oracle" / "_ref"
MODULES = ["param_fabric", "rng", "dataflow", "communicator", "migration", "cluster"]
KNOWN_REFERENCE_FAILURES = {
    "migration": {"stall dominance over fuzzed configurations", "byte-count law across D"},
}


def _run(binary: Path) -> str:
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=600)
    return r.stdout


def _normalise(out: str):
    cases = {}
    failures = []
    for line in out.splitlines():
        m = re.match(r"CASE (PASS|FAIL) (.*)", line)
        if m:
            cases[m.group(2)] = m.group(1)
        elif "failed" in line or "threw" in line:
            failures.append(line)
    return cases, failures


@pytest.mark.parametrize("module", MODULES)
def test_reference_unit_tests_identical(module):
    ref_bin = REF_DIR / f"test_{module}_ref"
    b200_bin = REF_DIR / f"test_{module}_b200"
    if not ref_bin.exists() or not b200_bin.exists():
        pytest.skip("reference test binaries not built (needs /root/reference; make -C oracle)")
    ref_cases, ref_fail = _normalise(_run(ref_bin))
    b200_cases, b200_fail = _normalise(_run(b200_bin))
    assert ref_cases and ref_cases == b200_cases
    assert ref_fail == b200_fail
    failed = {c for c, s in b200_cases.items() if s == "FAIL"}
    assert failed == KNOWN_REFERENCE_FAILURES.get(module, set())
