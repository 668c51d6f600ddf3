"""CPU cross-check of a document-KV blob the B200 path wrote (tests/golden/gpu_store,
made by tests/golden/make_gpu_blob.py on a GPU box):

* this package's KvStore finds it on disk and the native decode verifies its FNV-1a;
* the reference's own KvStore (ragdcache store.py:250-296, decode codec.py:282-295) reads
  the same file as a DISK_HIT with the same payload (the .rdkv written by the GPU
  generator is a valid reference blob, not just our noise blobs);
* the payload is the KV the fp32 oracle computes for the same tokens and weights
  (rel err <= 2e-2, the north-star bf16 bound).
"""
import json
import shutil
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
FIX = ROOT / "tests" / "golden" / "gpu_store"
pytestmark = pytest.mark.skipif(not (FIX / "fixture.json").exists(), reason="fixture not generated")


def _meta():
    return json.loads((FIX / "fixture.json").read_text())


def test_our_store_reads_gpu_blob(tmp_path):
    from paper_2504_11765_b200.store import KvKey, KvStore, Outcome

    m = _meta()
    root = tmp_path / "s"
    shutil.copytree(FIX, root)
    st = KvStore(root, memory_capacity_bytes=0)
    look = st.get(KvKey(m["model_hash"], tuple(m["doc_ids"])))
    assert look.outcome is Outcome.DISK_HIT
    assert look.blob.header.checksum == m["checksum"]
    assert look.blob.header.token_count == sum(m["doc_tokens"])


@pytest.mark.skipif(not Path("/root/reference/pkg/src").exists(), reason="reference not mounted (GPU box)")
def test_reference_store_reads_gpu_blob(tmp_path):
    sys.path.insert(0, "/root/reference/pkg/src")
    from ragdcache import store as rstore

    from paper_2504_11765_b200.store import KvKey, KvStore

    m = _meta()
    root = tmp_path / "s"
    shutil.copytree(FIX, root)
    ref = rstore.KvStore(root, memory_capacity_bytes=0)
    r = ref.get(rstore.KvKey(m["model_hash"], tuple(m["doc_ids"])))
    assert r.outcome is rstore.Outcome.DISK_HIT
    assert r.blob.header.checksum == m["checksum"]
    ours = KvStore(root, memory_capacity_bytes=0).get(KvKey(m["model_hash"], tuple(m["doc_ids"])))
    assert bytes(r.blob.payload) == bytes(ours.blob.payload_tensor().numpy().tobytes())


def test_gpu_blob_kv_matches_oracle():
    from oracle.llama_ref import OracleModel, rel_err
    from paper_2504_11765_b200.model import combo_tokens, get_spec, init_weights
    from paper_2504_11765_b200.store import KvKey, KvStore

    m = _meta()
    spec = get_spec(m["model"])
    w = init_weights(spec, m["seed"], device="cpu")
    # the engine folds the norm gains into w_qkv / w_gate_up (engine.fold_norm_gains): same here
    for lw in w.layers:
        for wk, gk in (("wqkv", "attn_norm"), ("wgu", "mlp_norm")):
            lw[wk] = (lw[wk].float() * lw[gk].float()[None, :]).to(lw[wk].dtype)
            lw[gk] = torch.ones_like(lw[gk])
    toks = combo_tokens(m["doc_ids"], m["doc_tokens"], spec.vocab)
    kv_ref, _ = OracleModel(w).forward(np.asarray(toks), want_logits=False)
    blob = KvStore(FIX, memory_capacity_bytes=0).get(KvKey(m["model_hash"], tuple(m["doc_ids"]))).blob
    n = sum(m["doc_tokens"])
    got = blob.payload_tensor().view(torch.bfloat16).view(spec.layers, 2, spec.kv_heads, n, spec.head_dim)
    assert rel_err(got, kv_ref) <= 2e-2
