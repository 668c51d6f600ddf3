"""K2/K4 attention kernels (rdkv_attention) against a plain PyTorch fp32
reference of the same op: causal GQA attention of the new tokens over the
cached prefix plus themselves (reference semantics: cached_prefill_work,
costs.py:89-99), KV read through a paged block table.

Tolerance: bf16 inputs/outputs, fp32 softmax/accumulation on both sides;
max|gpu - ref| <= 2e-2 * max|ref| (the north-star bf16 bound).
"""

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2504_11765_b200 import _lib

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _case(n_new, n_cached, hq, hkv, dh, block_size=64, seed=0, shuffle=True):
    g = torch.Generator().manual_seed(seed)
    S = len(n_new)
    ctx = [a + b for a, b in zip(n_new, n_cached)]
    nblk = [(c + block_size - 1) // block_size for c in ctx]
    total_blocks = sum(nblk) + 3
    perm = torch.randperm(total_blocks, generator=g) if shuffle else torch.arange(total_blocks)
    bt_stride = max(nblk)
    bt = torch.zeros(S, bt_stride, dtype=torch.int32)
    k = 0
    for s in range(S):
        bt[s, : nblk[s]] = perm[k: k + nblk[s]]
        k += nblk[s]
    slots = total_blocks * block_size
    kp = (torch.randn(hkv, slots, dh, generator=g)).bfloat16()
    vp = (torch.randn(hkv, slots, dh, generator=g)).bfloat16()
    T = sum(n_new)
    q = (torch.randn(T, hq * dh, generator=g) * 1.5).bfloat16()
    start = np.zeros(S, np.int32)
    start[1:] = np.cumsum(n_new)[:-1]
    return dict(q=q, kp=kp, vp=vp, bt=bt, slots=slots, start=torch.from_numpy(start),
                n_new=torch.tensor(n_new, dtype=torch.int32), n_cached=torch.tensor(n_cached, dtype=torch.int32),
                hq=hq, hkv=hkv, dh=dh, block_size=block_size, T=T, S=S)


def _reference(c):
    out = torch.zeros(c["T"], c["hq"] * c["dh"])
    G = c["hq"] // c["hkv"]
    dh, bs = c["dh"], c["block_size"]
    for s in range(c["S"]):
        nn, nc = int(c["n_new"][s]), int(c["n_cached"][s])
        L = nn + nc
        pos = torch.arange(L)
        slot = c["bt"][s, pos // bs].long() * bs + pos % bs
        K = c["kp"][:, slot].float()          # [hkv, L, dh]
        V = c["vp"][:, slot].float()
        a = int(c["start"][s])
        Q = c["q"][a: a + nn].float().view(nn, c["hq"], dh).transpose(0, 1)  # [hq, nn, dh]
        Kq = K.repeat_interleave(G, 0)
        Vq = V.repeat_interleave(G, 0)
        sc = Q @ Kq.transpose(1, 2) / dh ** 0.5
        qpos = torch.arange(nc, nc + nn)
        mask = pos[None, :] > qpos[:, None]
        sc = sc.masked_fill(mask[None], float("-inf"))
        o = torch.softmax(sc, -1) @ Vq                                       # [hq, nn, dh]
        out[a: a + nn] = o.transpose(0, 1).reshape(nn, -1)
    return out


def _run(c, impl, scratch=True):
    dev = "cuda"
    q, kp, vp = c["q"].to(dev), c["kp"].to(dev), c["vp"].to(dev)
    o = torch.full_like(q, float("nan"))
    bt = c["bt"].to(dev).contiguous()
    st, nn, nc = c["start"].to(dev), c["n_new"].to(dev), c["n_cached"].to(dev)
    lib = _lib.lib()
    ws = None
    nb = lib.rdkv_attention_scratch_bytes(c["T"], c["hq"], c["dh"])
    if scratch and nb:
        ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    max_ctx = int((c["n_new"] + c["n_cached"]).max())
    _lib.check(lib.rdkv_attention(
        _ptr(q), c["hq"] * c["dh"], _ptr(o), c["hq"] * c["dh"], _ptr(kp), _ptr(vp), c["slots"], _ptr(st), _ptr(nn),
        _ptr(nc), _ptr(bt), bt.shape[1], c["block_size"], c["S"], c["T"], int(c["n_new"].max()), max_ctx, c["hq"],
        c["hkv"], c["dh"], impl, _ptr(ws), nb if ws is not None else 0, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return o.float().cpu()


CASES = [
    # (n_new, n_cached, hq, hkv, dh)
    ([64], [2560], 32, 8, 64),                     # C2 query over a 5x512 composite
    ([64] * 4, [2560, 512, 1024, 0], 32, 8, 64),   # batch, ragged prefixes
    ([64, 17, 33, 1], [300, 1000, 0, 77], 32, 8, 128),   # C3 shape (dh 128), ragged both ways
    ([285], [0], 32, 8, 64),                       # document prefill (causal, no prefix)
    ([200, 96], [0, 128], 4, 4, 64),               # MHA (tiny model), G = 1
    ([40, 64], [640, 3], 64, 8, 128),              # G = 8 (70B shape)
    ([31], [5000], 32, 8, 128),                    # long prefix, single query
    ([1], [63], 8, 2, 64),                         # single token
]


@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("case", CASES, ids=[f"c{i}" for i in range(len(CASES))])
def test_attention_matches_torch_fp32(case, impl):
    c = _case(*case)
    got = _run(c, impl)
    ref = _reference(c)
    assert torch.isfinite(got).all()
    err = (got - ref).abs().max().item() / ref.abs().max().item()
    assert err <= TOL, f"rel err {err:.3e}"


def test_split_kv_equals_unsplit():
    # single sequence: the tcgen05 launcher splits the KV range when scratch is given
    c = _case([64], [4096], 32, 8, 64, seed=3)
    a = _run(c, 0, scratch=True)
    b = _run(c, 0, scratch=False)
    ref = _reference(c)
    assert (a - ref).abs().max() / ref.abs().max() <= TOL
    assert (a - b).abs().max() / ref.abs().max() <= 1e-2


def test_deterministic():
    c = _case([64] * 3, [2560, 100, 700], 32, 8, 64, seed=5)
    a = _run(c, 0)
    b = _run(c, 0)
    assert torch.equal(a, b)


def _ragged(S, seed, max_new=300, max_cached=3000):
    r = np.random.default_rng(seed)
    return [int(x) for x in r.integers(1, max_new, S)], [int(x) for x in r.integers(0, max_cached, S)]


# impl 2: grids of more than half a wave of (query block, kv head, sequence)
# units run stream-K: 148 persistent CTAs with equal KV-tile shares, units cut at
# share boundaries merged through (m, l, O) partials
SK_CASES = [
    ([64] * 32, [2560] * 32, 32, 8, 64),           # the C2 bench batch (256 units)
    (*_ragged(24, 1), 32, 8, 64),                  # ragged: multi-block queries, one-tile units
    ([64] * 16, [5120] * 16, 32, 8, 128),          # C3 batch (128 units on 148 SMs)
    ([64] * 12, [1000, 3, 2000, 64] * 3, 64, 8, 128),  # G = 8: two query blocks per query
    ([100] * 10, [50] * 10, 16, 16, 64),           # G = 1: one Q tile per unit
    (*_ragged(40, 2, max_new=70, max_cached=200), 32, 8, 64),  # many short units
]


@pytest.mark.parametrize("case", SK_CASES, ids=[f"sk{i}" for i in range(len(SK_CASES))])
def test_stream_k_matches_torch_fp32_and_per_unit_grid(case):
    c = _case(*case)
    got = _run(c, 2)
    ref = _reference(c)
    assert torch.isfinite(got).all()
    err = (got - ref).abs().max().item() / ref.abs().max().item()
    assert err <= TOL, f"rel err {err:.3e}"
    plain = _run(c, 0)  # one CTA per unit
    assert (got - plain).abs().max().item() / ref.abs().max().item() <= 1e-2
    assert torch.equal(got, _run(c, 2))  # same batch -> same shares -> same bits


# more than one wave with a mostly idle last wave: the sequences that fill whole waves
# run one CTA per unit, the rest split their KV range in 4 (+ combine)
TAIL_CASES = [
    ([64] * 24, [5120] * 24, 32, 8, 128),          # dh = 128: 192 units, 18 sequences whole, 6 split
    ([64] * 40, [4100] * 40, 32, 8, 64),           # dh = 64: 320 units of 33 KV tiles
    (*_ragged(30, 3, max_new=200, max_cached=6000), 32, 8, 64),
]


@pytest.mark.parametrize("case", TAIL_CASES, ids=[f"tail{i}" for i in range(len(TAIL_CASES))])
def test_tail_split_matches_torch_fp32_and_whole_units(case):
    c = _case(*case)
    got = _run(c, 0, scratch=True)
    ref = _reference(c)
    assert torch.isfinite(got).all()
    err = (got - ref).abs().max().item() / ref.abs().max().item()
    assert err <= TOL, f"rel err {err:.3e}"
    whole = _run(c, 0, scratch=False)
    assert (got - whole).abs().max().item() / ref.abs().max().item() <= 1e-2
    assert torch.equal(got, _run(c, 0, scratch=True))
