"""compute-sanitizer over every device kernel at small sizes
(scripts/sanitize_run.py): memcheck, synccheck and initcheck report no
errors.  racecheck is not asserted: it does not model mbarrier ordering and
reports the mbarrier-published shared-memory stores (profiles/r02_sanitizer.txt
lists and explains each one)."""
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "synccheck", "initcheck"])
def test_kernels_are_sanitizer_clean(tool):
    if not os.path.exists(SANITIZER):
        pytest.skip("compute-sanitizer not installed")
    # --num-cuda-barriers: the chain kernel's mbarriers outnumber synccheck's default tracking
    r = subprocess.run([SANITIZER, "--tool", tool, "--num-cuda-barriers", "256", "--error-exitcode", "3",
                        "--print-limit", "20", sys.executable, str(ROOT / "scripts" / "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert "sanitize_run done" in out, out[-3000:]
    assert r.returncode == 0 and "ERROR SUMMARY: 0 errors" in out, out[-3000:]
