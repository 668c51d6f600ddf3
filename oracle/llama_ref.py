"""fp32 PyTorch-CPU restatement of the hot path's numerics (TEST INFRASTRUCTURE).

Parity unpinned by the reference: ragdcache has no transformer;
its payloads are noise (codec.py:3-6) and prefill is a cost formula
(costs.py:82-99).  What the reference *does* pin, and what this module follows:

* a cache for the ordered combination [d1..dj] is the KV of those documents'
  concatenated tokens computed from scratch at positions 0..span-1
  (prefetch.py:6-8, :113-126; sim.py:487-490);
* with a cached prefix of n_cached tokens, only the new tokens (remaining
  documents, then the query: sim.py:420-422) are prefilled and they attend over
  the whole context (costs.py:3-7, :89-99); a miss prefills everything from raw
  text (costs.py:136-138);
* the first token is produced from the last position (costs.py:121-133).

The model is the Llama-shaped decoder described in paper_2504_11765_b200.model
(rotate-half RoPE, RMSNorm, GQA, SwiGLU); weights are the same bf16 tensors the
GPU uses, promoted to fp32.  Everything here runs in fp32 on the CPU.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def rope_tables(head_dim: int, theta: float, n_pos: int) -> tuple[torch.Tensor, torch.Tensor]:
    """cos/sin [n_pos, head_dim/2], computed in float64 and rounded once to fp32
    (the device table is built the same way)."""
    i = torch.arange(head_dim // 2, dtype=torch.float64)
    inv = torch.pow(torch.tensor(float(theta), dtype=torch.float64), -2.0 * i / head_dim)
    ang = torch.arange(n_pos, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.cos(ang).float(), torch.sin(ang).float()


def _rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    # x [n, H, dh]; cos/sin [n, dh/2]
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


def _rmsnorm(x: torch.Tensor, g: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


class OracleModel:
    """fp32 CPU copy of a ModelWeights."""

    def __init__(self, weights, n_threads: int | None = None) -> None:
        self.spec = s = weights.spec
        if n_threads:
            torch.set_num_threads(n_threads)
        f = lambda t: t.detach().to("cpu", torch.float32)
        self.embed = f(weights.embed)
        self.layers = []
        for i in range(s.layers):
            lw = weights.logical_layer(i)
            self.layers.append({k: f(v) for k, v in lw.items()})
        self.final_norm = f(weights.final_norm)
        self.lm_head = self.embed if s.tie_embeddings else f(weights.lm_head)

    @torch.no_grad()
    def forward(self, new_tokens, past_kv: torch.Tensor | None = None, n_cached: int = 0,
                want_logits: bool = True, layers: int | None = None):
        """Prefill ``new_tokens`` at positions [n_cached, n_cached + n) over a
        cached prefix ``past_kv`` [L][2][Hkv][n_cached][dh].

        Returns (kv [L][2][Hkv][n_cached + n][dh] fp32, logits [V] of the last
        position or None)."""
        s = self.spec
        L = s.layers if layers is None else layers
        tok = torch.as_tensor(new_tokens, dtype=torch.long)
        n = tok.numel()
        n_total = n_cached + n
        cos, sin = rope_tables(s.head_dim, s.rope_theta, n_total)
        cos, sin = cos[n_cached:], sin[n_cached:]
        x = self.embed[tok]
        kv_out = torch.empty(L, 2, s.kv_heads, n_total, s.head_dim)
        if n_cached:
            kv_out[:, :, :, :n_cached] = past_kv[:L].float()
        qpos = torch.arange(n_cached, n_total)
        kpos = torch.arange(n_total)
        mask = kpos[None, :] <= qpos[:, None]  # causal over the whole context
        scale = 1.0 / math.sqrt(s.head_dim)
        for li in range(L):
            w = self.layers[li]
            h = _rmsnorm(x, w["attn_norm"], s.norm_eps)
            q = (h @ w["wq"].T).view(n, s.n_heads, s.head_dim)
            k = (h @ w["wk"].T).view(n, s.kv_heads, s.head_dim)
            v = (h @ w["wv"].T).view(n, s.kv_heads, s.head_dim)
            q, k = _rope(q, cos, sin), _rope(k, cos, sin)
            kv_out[li, 0, :, n_cached:] = k.transpose(0, 1)
            kv_out[li, 1, :, n_cached:] = v.transpose(0, 1)
            K = kv_out[li, 0]  # [Hkv, n_total, dh]
            V = kv_out[li, 1]
            o = F.scaled_dot_product_attention(q.transpose(0, 1)[None], K[None], V[None], attn_mask=mask[None, None],
                                               scale=scale, enable_gqa=True)[0]
            x = x + o.transpose(0, 1).reshape(n, s.q_dim) @ w["wo"].T
            h = _rmsnorm(x, w["mlp_norm"], s.norm_eps)
            x = x + (F.silu(h @ w["wg"].T) * (h @ w["wu"].T)) @ w["wd"].T
        logits = None
        if want_logits:
            hl = _rmsnorm(x[-1], self.final_norm, s.norm_eps)
            logits = self.lm_head @ hl
        return kv_out, logits


def rel_err(a: torch.Tensor, b: torch.Tensor) -> float:
    """max |a - b| / max |b| — the tolerance metric of the parity tests."""
    a, b = a.float().cpu(), b.float().cpu()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def top1_margin(logits: torch.Tensor) -> float:
    t = torch.topk(logits.float(), 2).values
    return float(t[0] - t[1])
