"""Stream-K and B-multicast modes of the CTA-pair GEMM (RDKV_GEMM_SK, csrc/gemm_tc.cu launch_pair_auto)
against whole tiles on a 16-query C2 batch (M = 1024: gate/up = 256 tiles on 74 pairs, a
partial last round).  Split tiles only reorder the fp32 k-sum, so the logits agree to
fp32/bf16 rounding (rel err <= 2e-3) and the first tokens are identical."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _logits(tmp_path, mode, mc=0):
    out = tmp_path / f"sk{mode}_mc{mc}.npy"
    env = dict(os.environ, RDKV_GEMM_SK=str(mode), RDKV_GEMM_MC=str(mc))
    res = subprocess.run([sys.executable, str(ROOT / "scripts" / "sk_logits.py"), str(out)], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    return np.load(out)


@pytest.fixture(scope="module")
def whole_tiles(tmp_path_factory):
    return _logits(tmp_path_factory.mktemp("sk"), 0)


@pytest.mark.parametrize("mode", [2, 3])
def test_stream_k_modes_match_whole_tiles(tmp_path, whole_tiles, mode):
    base, got = whole_tiles, _logits(tmp_path, mode)
    assert base.shape == got.shape == (16, base.shape[1])
    err = np.abs(got - base).max() / np.abs(base).max()
    assert err <= 2e-3, f"rel err {err:.3e}"
    assert (got.argmax(1) == base.argmax(1)).all()


@pytest.mark.parametrize("mc", [1, 2])
def test_b_multicast_is_bit_exact(tmp_path, whole_tiles, mc):
    """RDKV_GEMM_MC: the B tile reaches both pairs of a cluster by TMA multicast; the MMAs and
    their k order are unchanged, so the logits are bit-identical."""
    got = _logits(tmp_path, 0, mc)
    assert np.array_equal(got, whole_tiles)
