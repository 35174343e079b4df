"""GPU: the small sanitizer workloads (scripts/sanitize_cases.py: every kernel family, counts and
tables checked against the oracle inside the run) through the bounds-checked build
(libdeltamotif_checked.so, DM_DCHECK device asserts on table / apex / pair indices).
compute-sanitizer is not available on the GPU pool, so the library checks its own indices."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_checked_build_runs_clean():
    lib = os.path.join(ROOT, "paper_2508_21287_b200", "libdeltamotif_checked.so")
    assert os.path.exists(lib), "build the checked variant: python -m paper_2508_21287_b200._build --checked"
    env = dict(os.environ, DM_LIBRARY_VARIANT="checked")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "sanitize cases ok" in r.stdout, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
