"""GPU: the reference's OWN test suite (225 tests of /root/reference/pkg/tests, copied
beside the reference install by __graft_entry__.build(), git-ignored) run with the seam
installed as a pytest plugin -- every forward / preprocess / linear_predict /
load_ensemble / apply_policy / gateway call those tests make goes through this package's
B200 path ("run the reference suite itself against the GPU path")."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("contexts", ["1", "3"])
def test_reference_suite_passes_through_the_seam(contexts):
    """(contexts = 3: three execution contexts per engine, so the suite's concurrent
    gateway tests run forwards in parallel on the GPU)"""
    suite = ROOT / "baseline" / "_ref_tests"
    ref = ROOT / "baseline" / "_ref"
    if not (suite / "conftest.py").exists() or not (ref / "ensemblegate").is_dir():
        pytest.fail("baseline/_ref(_tests) missing: run __graft_entry__.build() in the build container")
    env = dict(os.environ, PYTHONPATH=f"{ROOT}{os.pathsep}{ref}", PYTHONDONTWRITEBYTECODE="1",
               EB_CONTEXTS=contexts)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "-p", "paper_2003_01538_b200.seam", str(suite)],
                       cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=900)
    tail = r.stdout.strip().splitlines()[-3:]
    print("\n".join(tail))
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in tail[-1] and "failed" not in tail[-1]
