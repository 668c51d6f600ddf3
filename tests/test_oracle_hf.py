"""Pin the numerics oracle (oracle/llama_ref.py) to an independent Llama
implementation: HuggingFace transformers ``LlamaForCausalLM`` (fp32, eager),
run with the same weights by tests/golden/make_llama_golden.py.

The fixture pins the RoPE convention, RMSNorm placement, GQA mapping, SwiGLU,
tied embeddings and the cached-prefix (past_key_values) semantics.  Both sides
are fp32, so the bound is tight: max |oracle - hf| over the sampled entries and
projections <= 1e-4 of the tensor's max |value| (the only difference is the
RoPE angle table: float64 here, float32 in transformers).
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.llama_ref import OracleModel
from paper_2504_11765_b200.model import get_spec, init_weights

G = json.loads((Path(__file__).resolve().parent / "golden" / "llama_golden.json").read_text())
TOL = 1e-4


def _plan(shape, seed, n_sample, n_proj):
    n = int(np.prod(shape))
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=min(n_sample, n), replace=False))
    proj = rng.integers(0, 2, size=(n_proj, n)).astype(np.float64) * 2 - 1
    return idx, proj


def check_against(t: torch.Tensor, ref: dict, seed: int, tol: float, what: str) -> float:
    """Compare tensor ``t`` with a fixture summary; returns the worst relative error."""
    assert list(t.shape) == ref["shape"], (what, list(t.shape), ref["shape"])
    a = t.detach().double().reshape(-1).cpu().numpy()
    idx, proj = _plan(t.shape, seed, G["n_sample"], G["n_proj"])
    assert idx.tolist() == ref["idx"]
    scale = ref["max_abs"]
    err = np.abs(a[idx] - np.asarray(ref["val"])).max() / scale
    # projections sum n entries: bound by sqrt(n) * tol * scale
    perr = (np.abs(proj @ a - np.asarray(ref["proj"])) / (np.sqrt(a.size) * scale)).max()
    top = np.abs(a[ref["top_idx"]] - np.asarray(ref["top_val"])).max() / scale
    worst = float(max(err, perr, top))
    assert worst <= tol, f"{what}: rel err {worst:.3e} > {tol}"
    return worst


def weights_for(case, device="cpu"):
    spec = get_spec(case["spec"], case["layers"])
    w = init_weights(spec, seed=case["seed"], device="cpu")
    fp = case["weights"]
    l0 = w.layers[0]
    f = lambda t: float(t.detach().double().reshape(-1)[:4096].sum())
    got = {"embed": f(w.embed), "wqkv0": f(l0["wqkv"]), "wgu0": f(l0["wgu"]), "wdown0": f(l0["wdown"]),
           "final_norm": f(w.final_norm), "lm_head": f(w.lm_head)}
    for k, v in fp.items():
        assert abs(got[k] - v) <= 1e-9 * max(1.0, abs(v)), f"init_weights changed: {k}"
    return spec, w


@pytest.mark.parametrize("case", G["cases"], ids=lambda c: f"{c['spec']}@{c['layers']}L")
def test_oracle_matches_transformers_llama(case):
    spec, w = weights_for(case)
    orc = OracleModel(w)
    toks = np.asarray(case["tokens"], np.int32)
    n_pre = sum(case["doc_tokens"])
    from paper_2504_11765_b200.model import combo_tokens, query_tokens

    # the synthetic token streams are part of what is pinned
    assert toks[:n_pre].tolist() == combo_tokens(case["doc_ids"], case["doc_tokens"], spec.vocab).tolist()
    assert toks[n_pre:].tolist() == query_tokens(case["query_id"], case["query_tokens"], spec.vocab).tolist()
    kv_full, lg_full = orc.forward(toks)
    kv_pre, _ = orc.forward(toks[:n_pre], want_logits=False)
    _, lg_cached = orc.forward(toks[n_pre:], kv_pre, n_pre)
    check_against(kv_pre, case["kv_prefix"], 1, TOL, "prefix KV")
    check_against(kv_full, case["kv_full"], 2, TOL, "full KV")
    check_against(lg_full, case["logits_full"], 3, TOL, "full-prompt logits")
    check_against(lg_cached, case["logits_cached"], 4, TOL, "cached-prefix logits")
    assert int(torch.argmax(lg_full)) == case["logits_full"]["argmax"]
    assert int(torch.argmax(lg_cached)) == case["logits_cached"]["argmax"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", G["cases"], ids=lambda c: f"{c['spec']}@{c['layers']}L")
def test_device_path_matches_transformers_llama(case):
    """The product path (librdkv kernels) against the transformers fixture directly,
    at the north-star bf16 tolerance: document-KV generation, the query prefilled
    over the cached prefix, and the full-prompt (miss) prefill."""
    from paper_2504_11765_b200.engine import Engine, QueryRequest

    spec, w = weights_for(case)
    eng = Engine(spec, weights=w.to("cuda"), pool_tokens=4096)
    toks = np.asarray(case["tokens"], np.int32)
    n_pre = sum(case["doc_tokens"])
    kv = eng.generate_doc_kv(toks[:n_pre])
    lg_c, nx_c = eng.prefill([QueryRequest(toks[n_pre:], kv, n_pre)])
    lg_f, nx_f = eng.prefill([QueryRequest(toks)])
    torch.cuda.synchronize()
    kv = kv.view(spec.layers, 2, spec.kv_heads, n_pre, spec.head_dim).float().cpu()
    check_against(kv, case["kv_prefix"], 1, 2e-2, "device prefix KV")
    check_against(lg_c[0].cpu(), case["logits_cached"], 4, 2e-2, "device cached-prefix logits")
    check_against(lg_f[0].cpu(), case["logits_full"], 3, 2e-2, "device full-prompt logits")
    top = case["logits_cached"]
    margin = top["top_val"][0] - top["top_val"][1]
    err = float(np.abs(lg_c[0].double().cpu().numpy()[top["top_idx"]] - np.asarray(top["top_val"])).max())
    if margin > 2 * err:
        assert int(nx_c[0]) == top["argmax"] and int(nx_f[0]) == case["logits_full"]["argmax"]
