"""bench.py plumbing that runs without a GPU: the reference arm's JSON line (the
driver runs `bench.py --impl reference` beside our arm and computes the ratio),
the roofline inputs read from the committed profiles, and the config block."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_reference_arm_prints_the_contract_line():
    env = {**os.environ, "CUDA_VISIBLE_DEVICES": "", "OMP_NUM_THREADS": "2"}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--model", "tiny", "--steps", "2",
                        "--warmup", "1", "--k", "2", "--doc-tokens", "64", "--q-tokens", "16"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["unit"] == "queries/s" and line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "queries/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("C1 tiny-shaped")


def test_roofline_inputs_from_committed_profiles():
    peaks = bench._peaks()
    assert peaks["hbm_gbs"] > 1000 and peaks["bf16"] > 500
    for kernel in ("gemm_gate_up", "attention", "gemm_qkv", "gemm_o", "gemm_down"):
        t = bench._traffic_from_profiles(kernel)
        assert t is not None and t > 1e6, kernel
    assert bench._traffic_from_profiles("no_such_kernel") is None


@pytest.mark.parametrize("n", [1, 8])
def test_config_scales_global_batch(n):
    class A:
        model, k, doc_tokens, q_tokens, batch = "llama-3.2-1b", 5, 512, 64, 32
    c = bench._config(A, n)
    assert c["global_queries_per_step"] == 32 * n and c["cached_tokens_per_query"] == 2560
    assert c["parallelism"] == f"replicas x{n} (one instance per GPU)"
