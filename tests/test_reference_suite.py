"""Run the reference's OWN 78 unit/property tests against this package.

``holmes_planner`` is aliased to ``paper_2312_03549_b200`` and the reference
test files (/root/reference/pkg/tests, read-only, not copied) are executed
unchanged in a subprocess.  Only possible in the container that mounts the
reference; skipped elsewhere (the committed golden fixtures cover the GPU box).
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.reference
@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference not mounted")
def test_reference_unit_suite_passes_against_mirror(tmp_path):
    (tmp_path / "holmes_planner.py").write_text(
        "import sys\nimport paper_2312_03549_b200 as _m\nsys.modules[__name__] = _m\n")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(tmp_path), str(REF_TESTS), str(ROOT)])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "--rootdir", str(tmp_path), str(REF_TESTS)],
                       capture_output=True, text=True, env=env, cwd=tmp_path, timeout=300)
    tail = r.stdout[-4000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert "78 passed" in r.stdout, tail
