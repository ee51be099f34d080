"""compute-sanitizer memcheck over every kernel path (tools/sanitize_cases.py):
no out-of-bounds or misaligned accesses (sanitizers)."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_memcheck_clean():
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not available")
    r = subprocess.run([cs, "--tool", "memcheck", sys.executable, "tools/sanitize_cases.py"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert "sanitize cases done" in out, out[-2000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-2000:]
