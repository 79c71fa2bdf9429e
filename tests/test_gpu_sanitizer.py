"""compute-sanitizer memcheck / racecheck / synccheck over every kernel family (small grids,
including ragged extents, TMA-fed blocked kernels, reference kernels)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not available")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900)
    if "closed on this pool" in r.stdout + r.stderr:   # the GPU pool's wrapper refuses to run
        pytest.skip("compute-sanitizer is disabled on this GPU pool")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
