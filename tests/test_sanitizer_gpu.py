"""compute-sanitizer over the C1 hot path: memcheck (out-of-bounds /
misaligned device accesses, leaks of device allocations made by librdkv) and
racecheck (shared-memory hazards) on scripts/sanitize_c1.py.

Opt-in (RDKV_SANITIZE=1): the GPU pool has closed compute-sanitizer (runs under it left
GPUs needing a reset), so the suite does not launch it by default; the committed reports
are profiles/r2_sanitizer_*.txt and profiles/r2s3_sanitizer_*.txt."""

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
    if os.environ.get("RDKV_SANITIZE") != "1":
        pytest.skip("compute-sanitizer runs are opt-in (RDKV_SANITIZE=1)")
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, RDKV_PDL="0")  # the sanitizer serialises launches anyway
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20", sys.executable,
           str(ROOT / "scripts" / "sanitize_c1.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    out = res.stdout + res.stderr
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"sanitizer_{tool}.txt").write_text(out[-20000:])
    if "compute-sanitizer is closed" in out:
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert res.returncode == 0, out[-3000:]
    summary = "RACECHECK SUMMARY: 0 hazards displayed (0 errors" if tool == "racecheck" else "ERROR SUMMARY: 0 errors"
    assert summary in out, out[-3000:]
