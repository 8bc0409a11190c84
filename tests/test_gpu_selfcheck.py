"""compute-sanitizer is closed on the GPU pool; tools/selfcheck.py stands in for it
(bit-identical results over repeated launches of every kernel family = no
shared-memory / TMEM / barrier race observable; sentinel-filled padding and tails
around every output = no out-of-bounds write).  Run it in the GPU suite."""

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_selfcheck_repetition_and_guard_bands():
    res = subprocess.run([sys.executable, os.path.join(REPO, "tools", "selfcheck.py"), "3"],
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "SELF-CHECK PASSED" in res.stdout
