"""Drop-in check: the reference's OWN unit tests for the policy API
(pkg/tests/test_config.py, test_cache.py, test_cutoff.py) run unmodified
against this package through a ``moesim`` shim.  Needs /root/reference
(present in the build container only); skipped elsewhere."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = Path("/root/reference/pkg/tests")


@pytest.mark.parametrize("name", ["test_config.py", "test_cache.py", "test_cutoff.py"])
def test_reference_unit_tests_pass_against_b200_package(name, tmp_path):
    if not (REF_TESTS / name).exists():
        pytest.skip("reference tests not present on this machine")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "shim"), str(ROOT), str(REF_TESTS)])
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", str(tmp_path),
         "-c", os.devnull, str(REF_TESTS / name)],
        env=env, capture_output=True, text=True, cwd=tmp_path,
    )
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
