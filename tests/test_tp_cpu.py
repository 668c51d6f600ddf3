"""Tensor-parallel weight sharding (model.shard_weights) on CPU: the shards of
T ranks partition the heads and FFN columns exactly, so column-parallel
projections concatenate and row-parallel ones sum back to the full layer."""

import pytest
import torch

from paper_2504_11765_b200.model import get_spec, init_weights, shard_weights, tp_spec


@pytest.mark.parametrize("world", [2, 4])
def test_shards_reconstruct_the_layer(world):
    spec = get_spec("gqa-tp")
    full = init_weights(spec, seed=1, device="cpu")
    shards = [shard_weights(full, r, world) for r in range(world)]
    ls = tp_spec(spec, world)
    assert all(s.spec == ls for s in shards)
    g = torch.Generator().manual_seed(0)
    x = torch.randn(5, spec.hidden, generator=g)
    for li in range(spec.layers):
        F = full.logical_layer(li)
        parts = [s.logical_layer(li) for s in shards]
        for name in ("wq", "wk", "wv", "wg", "wu"):   # column-parallel: outputs concatenate
            got = torch.cat([x @ p[name].float().T for p in parts], dim=1)
            assert torch.allclose(got, x @ F[name].float().T, atol=1e-4), name
        # row-parallel: each rank's input slice times its columns sums to the full output
        a = torch.randn(5, spec.q_dim, generator=g)
        hq = ls.q_dim
        got = sum(a[:, r * hq:(r + 1) * hq] @ parts[r]["wo"].float().T for r in range(world))
        assert torch.allclose(got, a @ F["wo"].float().T, atol=1e-3)
        h = torch.randn(5, spec.ffn, generator=g)
        f = ls.ffn
        got = sum(h[:, r * f:(r + 1) * f] @ parts[r]["wd"].float().T for r in range(world))
        assert torch.allclose(got, h @ F["wd"].float().T, atol=1e-3)


def test_unshardable_shape_rejected():
    with pytest.raises(ValueError):
        tp_spec(get_spec("gqa-small-64"), 4)    # 2 KV heads cannot split 4 ways
    assert tp_spec(get_spec("llama-3-70b"), 4).kv_heads == 2
