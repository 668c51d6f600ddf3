"""Independent pin for the numerics oracle: HuggingFace ``LlamaForCausalLM``.

The reference (ragdcache) has no model, so ``oracle/llama_ref.py`` cannot be
checked against it.  This script runs the *transformers* Llama implementation
(5.5.0, fp32 on the CPU, eager attention) with exactly the weights
``paper_2504_11765_b200.model.init_weights(spec, seed, "cpu")`` produces and
records samples of what it computes:

* the K (post-RoPE) / V cache of a document prefix (``past_key_values``),
* the last-position logits of the full prompt (prefix + query),
* the last-position logits of the query prefilled over the cached prefix
  (``past_key_values`` fed back: the cached-prefix semantics of
  costs.py:89-99 / PAPER.md:165-166),

which pins the RoPE convention (rotate-half, theta, no scaling), RMSNorm
placement and epsilon, the GQA head mapping, SwiGLU and tied embeddings.
Shapes: C1 tiny (full), Llama-3.2-1B and Llama-3-8B at full width with 2
layers, and the dh=128 GQA test shape.  Output: ``llama_golden.json`` (samples
+ projections, not full tensors, so the fixture stays small).

    python tests/golden/make_llama_golden.py      # ~2 min, needs transformers
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2504_11765_b200.model import combo_tokens, get_spec, init_weights, query_tokens  # noqa: E402

OUT = Path(__file__).resolve().parent / "llama_golden.json"

# (spec, layers, weight seed, doc ids, doc token counts, query id, query tokens)
CASES = [
    ("tiny", None, 0, (3, 8), (96, 64), 1, 32),
    ("gqa-small-128", None, 2, (5, 9, 2), (128, 100, 61), 7, 24),
    ("llama-3.2-1b", 2, 0, (11, 4), (160, 96), 3, 40),
    ("llama-3-8b", 2, 0, (21, 22), (128, 100), 5, 40),
]
N_SAMPLE = 256
N_PROJ = 4


def sample_plan(shape, seed):
    """Fixed random flat indices + +-1 projection vectors for a tensor shape."""
    n = int(np.prod(shape))
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=min(N_SAMPLE, n), replace=False))
    proj = rng.integers(0, 2, size=(N_PROJ, n)).astype(np.float64) * 2 - 1
    return idx, proj


def summarize(t: torch.Tensor, seed: int) -> dict:
    a = t.detach().double().reshape(-1).numpy()
    idx, proj = sample_plan(t.shape, seed)
    top = np.argsort(a)[-16:][::-1]
    return {"shape": list(t.shape), "max_abs": float(np.abs(a).max()), "idx": idx.tolist(),
            "val": a[idx].tolist(), "proj": (proj @ a).tolist(), "top_idx": top.tolist(),
            "top_val": a[top].tolist(), "argmax": int(a.argmax())}


def weight_fingerprint(w) -> dict:
    f = lambda t: float(t.detach().double().reshape(-1)[:4096].sum())
    l0 = w.layers[0]
    return {"embed": f(w.embed), "wqkv0": f(l0["wqkv"]), "wgu0": f(l0["wgu"]), "wdown0": f(l0["wdown"]),
            "final_norm": f(w.final_norm), "lm_head": f(w.lm_head)}


def hf_model(w):
    from transformers import LlamaConfig, LlamaForCausalLM

    s = w.spec
    cfg = LlamaConfig(vocab_size=s.vocab, hidden_size=s.hidden, intermediate_size=s.ffn, num_hidden_layers=s.layers,
                      num_attention_heads=s.n_heads, num_key_value_heads=s.kv_heads, head_dim=s.head_dim,
                      rope_theta=s.rope_theta, rms_norm_eps=s.norm_eps, max_position_embeddings=s.max_pos,
                      tie_word_embeddings=s.tie_embeddings, attention_bias=False, mlp_bias=False,
                      attn_implementation="eager")
    m = LlamaForCausalLM(cfg).float().eval()
    f = lambda t: t.detach().float().clone()
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(f(w.embed))
        for i, layer in enumerate(m.model.layers):
            lw = w.logical_layer(i)
            a = layer.self_attn
            a.q_proj.weight.copy_(f(lw["wq"]))
            a.k_proj.weight.copy_(f(lw["wk"]))
            a.v_proj.weight.copy_(f(lw["wv"]))
            a.o_proj.weight.copy_(f(lw["wo"]))
            layer.mlp.gate_proj.weight.copy_(f(lw["wg"]))
            layer.mlp.up_proj.weight.copy_(f(lw["wu"]))
            layer.mlp.down_proj.weight.copy_(f(lw["wd"]))
            layer.input_layernorm.weight.copy_(f(lw["attn_norm"]))
            layer.post_attention_layernorm.weight.copy_(f(lw["mlp_norm"]))
        m.model.norm.weight.copy_(f(w.final_norm))
        if not s.tie_embeddings:
            m.lm_head.weight.copy_(f(w.lm_head))
    if s.tie_embeddings:
        assert m.lm_head.weight.data_ptr() == m.model.embed_tokens.weight.data_ptr()
    return m


def kv_stack(cache, n_layers: int) -> torch.Tensor:
    """HF cache -> [L][2][Hkv][n][dh] (our payload layout)."""
    out = []
    for li in range(n_layers):
        lay = cache.layers[li]
        out.append(torch.stack([lay.keys[0], lay.values[0]]))
    return torch.stack(out)


@torch.no_grad()
def run_case(name, layers, seed, docs, counts, qid, qn) -> dict:
    spec = get_spec(name, layers)
    w = init_weights(spec, seed=seed, device="cpu")
    m = hf_model(w)
    prefix = combo_tokens(docs, counts, spec.vocab)
    q = query_tokens(qid, qn, spec.vocab)
    full = torch.from_numpy(np.concatenate([prefix, q]).astype(np.int64))[None]
    out_full = m(full, use_cache=True, logits_to_keep=1)
    out_pre = m(full[:, : len(prefix)], use_cache=True, logits_to_keep=1)
    kv_prefix = kv_stack(out_pre.past_key_values, spec.layers)
    out_q = m(full[:, len(prefix):], past_key_values=out_pre.past_key_values, use_cache=True, logits_to_keep=1)
    kv_all = kv_stack(out_full.past_key_values, spec.layers)
    return {
        "spec": name, "layers": spec.layers, "seed": seed, "doc_ids": list(docs), "doc_tokens": list(counts),
        "query_id": qid, "query_tokens": qn, "tokens": full[0].tolist(),
        "weights": weight_fingerprint(w),
        "kv_prefix": summarize(kv_prefix, 1), "kv_full": summarize(kv_all, 2),
        "logits_full": summarize(out_full.logits[0, -1], 3),
        "logits_cached": summarize(out_q.logits[0, -1], 4),
    }


def main() -> None:
    import transformers

    torch.manual_seed(0)
    cases = []
    for c in CASES:
        r = run_case(*c)
        print(f"{r['spec']}@{r['layers']}L: argmax full {r['logits_full']['argmax']} "
              f"cached {r['logits_cached']['argmax']}", flush=True)
        cases.append(r)
    OUT.write_text(json.dumps({"generator": f"transformers {transformers.__version__} LlamaForCausalLM fp32 eager",
                               "n_sample": N_SAMPLE, "n_proj": N_PROJ, "cases": cases}))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
