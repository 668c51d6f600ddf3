"""CPU checks of the numerics oracle and the host-side model plumbing (no GPU)."""

import numpy as np
import torch

from oracle.llama_ref import OracleModel, rel_err
from paper_2504_11765_b200.engine import BatchPlan, SeqPlan
from paper_2504_11765_b200.model import SPECS, combo_tokens, doc_tokens, get_spec, init_weights, query_tokens


def _orc(name="gqa-small-64"):
    spec = get_spec(name)
    return spec, OracleModel(init_weights(spec, seed=3, device="cpu"))


def test_oracle_cached_prefix_equals_full_prompt():
    """Prefix semantics (costs.py:89-99): prefilling new tokens over the cached KV
    of the prefix gives the same logits as prefilling the whole prompt."""
    spec, orc = _orc()
    pre = combo_tokens([1, 2], [40, 23], spec.vocab)
    new = query_tokens(5, 17, spec.vocab)
    kv, _ = orc.forward(pre, want_logits=False)
    kv2, lg_cached = orc.forward(new, kv, len(pre))
    kvf, lg_full = orc.forward(np.concatenate([pre, new]))
    assert rel_err(lg_cached, lg_full) < 1e-4
    assert rel_err(kv2, kvf) < 1e-4


def test_oracle_prefix_kv_is_a_prefix():
    """KV of combination [d1..dj] = the first rows of the KV of [d1..dk] (causality);
    this is what makes single-pass prefix generation possible (SURVEY H-e)."""
    spec, orc = _orc("gqa-small-128")
    toks = combo_tokens([4, 8, 15], [30, 30, 30], spec.vocab)
    kv_all, _ = orc.forward(toks, want_logits=False)
    kv_2, _ = orc.forward(toks[:60], want_logits=False)
    assert rel_err(kv_all[:, :, :, :60], kv_2) < 1e-5


def test_tokens_deterministic_and_order_significant():
    a = combo_tokens([2, 1], [8, 8], 1000)
    b = combo_tokens([1, 2], [8, 8], 1000)
    assert not np.array_equal(a, b)
    assert np.array_equal(doc_tokens(7, 16, 5000), doc_tokens(7, 16, 5000))
    assert doc_tokens(7, 16, 5000).max() < 5000


def test_batch_plan_slots_and_positions():
    seqs = [SeqPlan(np.arange(10, dtype=np.int32), 70, [5, 2]), SeqPlan(np.arange(3, dtype=np.int32), 0, [9])]
    p = BatchPlan(seqs, block_size=64, device="cpu")
    m = p.meta.numpy()
    T = 13
    pos, slot = m[T:2 * T], m[2 * T:3 * T]
    assert list(pos[:10]) == list(range(70, 80)) and list(pos[10:]) == [0, 1, 2]
    assert list(slot[:10]) == [2 * 64 + (70 - 64) + i for i in range(10)]
    assert list(slot[10:]) == [9 * 64 + i for i in range(3)]
    assert p.max_new == 10 and p.bt_stride == 2


def test_spec_flops_and_profiles():
    s = SPECS["llama-3.2-1b"]
    assert s.profile().hidden_dim == 512 and s.profile().model_id == "llama-3.2-1b/bf16"
    assert s.kv_bytes_per_token() == 32 * 1024
    assert abs(s.prefill_flops(64, 2560) / 1e12 - 0.147) < 0.005
