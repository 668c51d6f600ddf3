"""compute-sanitizer over the C1 hot path: memcheck (out-of-bounds /
misaligned device accesses, leaks of device allocations made by librdkv) and
racecheck (shared-memory hazards) on scripts/sanitize_c1.py."""

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_c1_hot_path_is_sanitizer_clean(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, RDKV_PDL="0")  # the sanitizer serialises launches anyway
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20", sys.executable,
           str(ROOT / "scripts" / "sanitize_c1.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    out = res.stdout + res.stderr
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"sanitizer_{tool}.txt").write_text(out[-20000:])
    assert res.returncode == 0, out[-3000:]
    summary = "RACECHECK SUMMARY: 0 hazards displayed (0 errors" if tool == "racecheck" else "ERROR SUMMARY: 0 errors"
    assert summary in out, out[-3000:]
