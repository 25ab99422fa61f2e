"""Pin the planner oracle: oracle/_ref is the UNMODIFIED reference built by
oracle/Makefile; its own doctest suites and acceptance binary must pass
(85 cases, 10 criteria) before its outputs are trusted as golden fixtures."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref")
SUITES = ["test_trace", "test_hardware", "test_layout", "test_presets", "test_cost", "test_sim",
          "test_search", "test_cli"]


def _bin(name):
    p = os.path.join(REF, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (make -C oracle ref needs /root/reference)")
    return p


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes(suite, tmp_path):
    r = subprocess.run([_bin(suite)], cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_reference_acceptance_passes(tmp_path):
    r = subprocess.run([_bin("acceptance")], cwd=tmp_path, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.count("[PASS]") == 10, r.stdout
