"""compute-sanitizer over the device loop: memcheck,
racecheck and synccheck on small solves that exercise the fused controllers
(last-CTA tickets with __threadfence), the PDL step launches, the cone-block
classes (SOC half-warp, exp thread-per-block) and the check path (metrics,
rays, batched gap probes, restarts).  Each run must report 0 errors."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("case", ["c1s", "c2s", "c3s"])
def test_sanitizer_clean(tool, case):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "17", "--target-processes", "all",
           sys.executable, os.path.join(REPO, "tools", "sanitize_case.py"), case, "300"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    out = res.stdout + res.stderr
    if "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses every run (it has
        # left GPUs needing a reset); tests/test_gpu_bounds.py is the stand-in
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert res.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
    assert f"{case}:" in out, out[-2000:]
