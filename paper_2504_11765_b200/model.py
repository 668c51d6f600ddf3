"""Model shapes, seeded random-init weights and synthetic token streams.

The reference has no model: prefill is the analytic ``layers * n^2 * hidden``
(costs.py:82-99) and KV payloads are noise (codec.py:188-224).  The B200 build
runs a real Llama-shaped decoder (RMSNorm, rotate-half RoPE, grouped-query
attention, SwiGLU) with random-init weights of the shapes BASELINE.json names.
Document tokens are synthesised deterministically per doc id (the reference has
no text: workload.py:28-47), which keeps ``generate()`` deterministic per key as
service.py:92 requires.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np
import torch

from .codec import ModelProfile, splitmix64, splitmix_words

_U64 = (1 << 64) - 1


@dataclass(frozen=True)
class ModelSpec:
    name: str
    layers: int
    hidden: int
    n_heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    max_pos: int = 32768
    tie_embeddings: bool = False

    @property
    def q_dim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def qkv_rows(self) -> int:
        return (self.n_heads + 2 * self.kv_heads) * self.head_dim

    def profile(self) -> ModelProfile:
        """KV-size profile for the store.  GQA models use hidden_dim := kv_heads*head_dim
        (the only value codec.py:89-93 accepts); the dtype lives in the id so
        bf16/fp16 blobs never collide (SURVEY H-b)."""
        return ModelProfile(f"{self.name}/bf16", self.layers, self.kv_heads * self.head_dim, self.kv_heads,
                            self.head_dim, 2)

    def kv_bytes_per_token(self) -> int:
        return 2 * self.layers * self.kv_heads * self.head_dim * 2

    def nonembedding_params(self) -> int:
        per_layer = self.hidden * self.qkv_rows + self.q_dim * self.hidden + 3 * self.hidden * self.ffn
        return self.layers * per_layer

    def prefill_flops(self, n_new: int, n_cached: int = 0, with_head: bool = True) -> float:
        """Algorithmic FLOPs of prefilling n_new tokens after n_cached cached ones
        (GEMMs + causal attention score/value products + last-row LM head)."""
        gemm = 2.0 * self.nonembedding_params() * n_new
        # new token i (0-based) attends over n_cached + i + 1 positions
        ctx = n_new * n_cached + n_new * (n_new + 1) / 2.0
        attn = 4.0 * self.q_dim * ctx * self.layers
        head = 2.0 * self.hidden * self.vocab if with_head else 0.0
        return gemm + attn + head


SPECS: dict[str, ModelSpec] = {
    # C1: BASELINE configs[0], CPU-checkable
    "tiny": ModelSpec("tiny", layers=2, hidden=256, n_heads=4, kv_heads=4, head_dim=64, ffn=768, vocab=32000,
                      rope_theta=10000.0, max_pos=4096),
    # C2: Llama-3.2-1B-shaped (tied embeddings, like the real model)
    "llama-3.2-1b": ModelSpec("llama-3.2-1b", layers=16, hidden=2048, n_heads=32, kv_heads=8, head_dim=64,
                              ffn=8192, vocab=128256, tie_embeddings=True),
    # C3/C4: Llama-3-8B-shaped
    "llama-3-8b": ModelSpec("llama-3-8b", layers=32, hidden=4096, n_heads=32, kv_heads=8, head_dim=128,
                            ffn=14336, vocab=128256),
    # C5: Llama-3-70B-shaped (single-instance parity runs use a layer-truncated copy)
    "llama-3-70b": ModelSpec("llama-3-70b", layers=80, hidden=8192, n_heads=64, kv_heads=8, head_dim=128,
                             ffn=28672, vocab=128256),
    # small GQA shapes used by the parity tests (exercise dh=64 and dh=128 with groups)
    "gqa-small-64": ModelSpec("gqa-small-64", layers=2, hidden=512, n_heads=8, kv_heads=2, head_dim=64, ffn=1024,
                              vocab=4096, max_pos=8192),
    "gqa-small-128": ModelSpec("gqa-small-128", layers=2, hidden=1024, n_heads=8, kv_heads=2, head_dim=128,
                               ffn=2048, vocab=8192, max_pos=8192),
    # tensor-parallel parity shape: shards 2 and 4 ways (GQA group 2 per rank)
    "gqa-tp": ModelSpec("gqa-tp", layers=2, hidden=1024, n_heads=16, kv_heads=8, head_dim=64, ffn=2048,
                        vocab=4096, max_pos=8192),
}


def tp_spec(spec: ModelSpec, size: int) -> ModelSpec:
    """The per-rank shape of a tensor-parallel group of ``size`` ranks: 1/size of
    the query heads, KV heads and FFN columns (hidden, vocab replicated)."""
    if spec.n_heads % size or spec.kv_heads % size or spec.ffn % (64 * size):
        raise ValueError(f"{spec.name} does not shard {size} ways")
    return replace(spec, n_heads=spec.n_heads // size, kv_heads=spec.kv_heads // size, ffn=spec.ffn // size)


def shard_weights(w: "ModelWeights", rank: int, size: int) -> "ModelWeights":
    """Rank ``rank``'s shard of full weights: column-parallel wqkv (its query /
    key / value heads) and w_gate_up (its 64-row gate/up blocks), row-parallel
    wo and w_down (matching input columns).  Embedding, norms and LM head are
    replicated (shared tensors)."""
    s = w.spec
    ls = tp_spec(s, size)
    d, dh = s.hidden, s.head_dim
    hq, hk, f = ls.n_heads, ls.kv_heads, ls.ffn
    out = ModelWeights(spec=ls, embed=w.embed, final_norm=w.final_norm, lm_head=w.lm_head)
    for lw in w.layers:
        q, k = s.q_dim, s.kv_heads * dh
        wq = lw["wqkv"][:q].view(s.n_heads, dh, d)[rank * hq:(rank + 1) * hq].reshape(-1, d)
        wk = lw["wqkv"][q:q + k].view(s.kv_heads, dh, d)[rank * hk:(rank + 1) * hk].reshape(-1, d)
        wv = lw["wqkv"][q + k:].view(s.kv_heads, dh, d)[rank * hk:(rank + 1) * hk].reshape(-1, d)
        blocks = lw["wgu"].view(s.ffn // 64, 2 * 64, d)[rank * (f // 64):(rank + 1) * (f // 64)]
        out.layers.append({
            "attn_norm": lw["attn_norm"], "mlp_norm": lw["mlp_norm"],
            "wqkv": torch.cat([wq, wk, wv]).contiguous(),
            "wo": lw["wo"][:, rank * hq * dh:(rank + 1) * hq * dh].contiguous(),
            "wgu": blocks.reshape(2 * f, d).clone(),  # own storage: a shard's norm-gain fold stays in the shard
            "wdown": lw["wdown"][:, rank * f:(rank + 1) * f].contiguous(),
        })
    return out


def get_spec(name: str, layers: int | None = None) -> ModelSpec:
    spec = SPECS[name]
    return replace(spec, layers=layers) if layers is not None else spec


@dataclass
class ModelWeights:
    """bf16 weights (fp32 norm gains) in the device packing of include/rdkv.h."""

    spec: ModelSpec
    embed: torch.Tensor                    # [V, d]
    layers: list[dict] = field(default_factory=list)  # attn_norm, wqkv, wo, mlp_norm, wgu, wdown
    final_norm: torch.Tensor | None = None
    lm_head: torch.Tensor | None = None

    def pointer_list(self) -> list[int]:
        ptrs = [self.embed.data_ptr()]
        for lw in self.layers:
            ptrs += [lw[k].data_ptr() for k in ("attn_norm", "wqkv", "wo", "mlp_norm", "wgu", "wdown")]
        ptrs += [self.final_norm.data_ptr(), self.lm_head.data_ptr()]
        return ptrs

    def to(self, device) -> "ModelWeights":
        """Copy on ``device`` (tied embeddings stay tied)."""
        mv = lambda t: t.to(device)
        out = ModelWeights(spec=self.spec, embed=mv(self.embed), final_norm=mv(self.final_norm))
        out.lm_head = out.embed if self.lm_head is self.embed else mv(self.lm_head)
        out.layers = [{k: mv(v) for k, v in lw.items()} for lw in self.layers]
        return out

    # logical (unpacked) views for the oracle -----------------------------------
    def logical_layer(self, i: int) -> dict:
        s = self.spec
        lw = self.layers[i]
        q, k = s.q_dim, s.kv_heads * s.head_dim
        gu = lw["wgu"].view(s.ffn // 64, 2, 64, s.hidden)
        return {
            "attn_norm": lw["attn_norm"], "mlp_norm": lw["mlp_norm"],
            "wq": lw["wqkv"][:q], "wk": lw["wqkv"][q:q + k], "wv": lw["wqkv"][q + k:],
            "wo": lw["wo"], "wg": gu[:, 0].reshape(s.ffn, s.hidden), "wu": gu[:, 1].reshape(s.ffn, s.hidden),
            "wd": lw["wdown"],
        }


def init_weights(spec: ModelSpec, seed: int = 0, device: str | torch.device = "cuda") -> ModelWeights:
    """Seeded normal(0, sigma) init, cast to bf16.  Scales keep the
    residual stream O(1): projections 1/sqrt(fan_in), output projections an
    extra 1/sqrt(2L), LM head 1/sqrt(d) so logits are ~N(0, 1)."""
    g = torch.Generator(device=device).manual_seed(seed)
    d, L = spec.hidden, spec.layers

    def normal(shape, std):
        return (torch.randn(shape, generator=g, device=device, dtype=torch.float32) * std).to(torch.bfloat16)

    def gain():
        return 1.0 + 0.05 * torch.randn(d, generator=g, device=device, dtype=torch.float32)

    w = ModelWeights(spec=spec, embed=normal((spec.vocab, d), 1.0))
    out_scale = 1.0 / (2 * L) ** 0.5
    for _ in range(L):
        w.layers.append({
            "attn_norm": gain(),
            "wqkv": normal((spec.qkv_rows, d), d ** -0.5),
            "wo": normal((d, spec.q_dim), spec.q_dim ** -0.5 * out_scale),
            "mlp_norm": gain(),
            "wgu": normal((2 * spec.ffn, d), d ** -0.5),
            "wdown": normal((d, spec.ffn), spec.ffn ** -0.5 * out_scale),
        })
    w.final_norm = gain()
    w.lm_head = w.embed if spec.tie_embeddings else normal((spec.vocab, d), d ** -0.5)
    return w


# ----------------------------------------------------------------- synthetic tokens

_DOC_DOMAIN = 0xD0C5D0C5D0C5D0C5
_QUERY_DOMAIN = 0x0E3E0E3E0E3E0E3E


def doc_tokens(doc_id: int, n: int, vocab: int, seed: int = 0) -> np.ndarray:
    """Deterministic token ids of document ``doc_id`` (splitmix64 stream mod vocab)."""
    state = splitmix64(splitmix64((seed & _U64) ^ _DOC_DOMAIN) ^ (int(doc_id) & _U64))
    return (splitmix_words(state, n) % np.uint64(vocab)).astype(np.int32)


def query_tokens(query_id: int, n: int, vocab: int, seed: int = 0) -> np.ndarray:
    state = splitmix64(splitmix64((seed & _U64) ^ _QUERY_DOMAIN) ^ (int(query_id) & _U64))
    return (splitmix_words(state, n) % np.uint64(vocab)).astype(np.int32)


def combo_tokens(doc_ids, doc_token_counts, vocab: int, seed: int = 0) -> np.ndarray:
    """Concatenated tokens of an ordered document combination (prefetch.py:6-8)."""
    parts = [doc_tokens(d, n, vocab, seed) for d, n in zip(doc_ids, doc_token_counts)]
    return np.concatenate(parts) if parts else np.zeros(0, np.int32)
