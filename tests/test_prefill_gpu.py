"""Device path parity: document-KV generation, K3 unpack and cached-prefix
query prefill through librdkv, against the fp32 CPU oracle.

Tolerance (stated per north_star): rel err = max|gpu - oracle| / max|oracle|
<= 2e-2 for KV tensors and logits; first-token argmax identical whenever the
oracle's top-1 margin exceeds 4x the observed logit error (random-init logits
can nearly tie, SURVEY H-h); bit-exact for the integer/byte work (unpack).
"""

import numpy as np
import pytest
import torch

from oracle.llama_ref import OracleModel, rel_err, top1_margin
from paper_2504_11765_b200.engine import Engine, KvPool, QueryRequest, kv_unpack
from paper_2504_11765_b200.model import combo_tokens, get_spec, query_tokens

pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module", params=["tiny", "gqa-small-64", "gqa-small-128"])
def setup(request):
    spec = get_spec(request.param)
    eng = Engine(spec, seed=1, pool_tokens=16384, block_size=64)
    orc = OracleModel(eng.weights)
    return spec, eng, orc


def _kv_view(spec, flat, n):
    return flat.view(spec.layers, 2, spec.kv_heads, n, spec.head_dim)


def _check_logits(gpu_logits, ref_logits, gpu_arg):
    err = rel_err(gpu_logits, ref_logits)
    assert err <= TOL, f"logits rel err {err:.3e}"
    abs_err = float((gpu_logits.float().cpu() - ref_logits).abs().max())
    if top1_margin(ref_logits) > 4 * abs_err:
        assert int(gpu_arg) == int(torch.argmax(ref_logits))


def test_doc_prefill_kv_matches_oracle(setup):
    spec, eng, orc = setup
    toks = combo_tokens([7, 3, 11], [128, 96, 61], spec.vocab)  # ragged: 285 tokens
    kv = eng.generate_doc_kv(toks)
    torch.cuda.synchronize()
    ref, _ = orc.forward(toks, want_logits=False)
    got = _kv_view(spec, kv, len(toks)).float().cpu()
    assert torch.isfinite(got).all()
    assert rel_err(got, ref) <= TOL, rel_err(got, ref)


def test_cached_prefix_query_matches_full_prompt(setup):
    spec, eng, orc = setup
    docs, ntok = [5, 9, 2], [128, 128, 100]
    prefix = combo_tokens(docs[:2], ntok[:2], spec.vocab)            # cached: prefix j=2
    rest = np.concatenate([combo_tokens(docs[2:], ntok[2:], spec.vocab), query_tokens(1, 32, spec.vocab)])
    cached = eng.generate_doc_kv(prefix)
    logits, nxt = eng.prefill([QueryRequest(rest, cached, len(prefix))])
    # full prompt on the GPU (n_cached = 0): the miss path of costs.ttft
    full_logits, full_nxt = eng.prefill([QueryRequest(np.concatenate([prefix, rest]))])
    torch.cuda.synchronize()
    _, ref = orc.forward(np.concatenate([prefix, rest]))
    _check_logits(logits[0], ref, nxt[0])
    _check_logits(full_logits[0], ref, full_nxt[0])
    assert rel_err(logits[0], full_logits[0]) <= TOL


def test_long_cached_prefix_split_kv(setup):
    """A single query over a long cached prefix: the grid is tiny, so the
    tensor-core attention splits the KV range across CTAs and merges partials."""
    spec, eng, orc = setup
    prefix = combo_tokens([21, 22, 23], [512, 512, 476], spec.vocab)    # 1500 cached tokens
    new = query_tokens(9, 40, spec.vocab)
    cached = eng.generate_doc_kv(prefix)
    logits, nxt = eng.prefill([QueryRequest(new, cached, len(prefix))])
    torch.cuda.synchronize()
    _, ref = orc.forward(np.concatenate([prefix, new]))
    _check_logits(logits[0], ref, nxt[0])


def test_batched_ragged_equals_single(setup):
    spec, eng, orc = setup
    reqs, singles = [], []
    for i, (nc, nn) in enumerate([(0, 40), (128, 64), (200, 17), (64, 130)]):
        pre = combo_tokens([100 + i], [nc], spec.vocab) if nc else None
        new = query_tokens(50 + i, nn, spec.vocab)
        cached = eng.generate_doc_kv(pre) if nc else None
        reqs.append(QueryRequest(new, cached, nc))
    lb, nb = eng.prefill(reqs)
    for i, r in enumerate(reqs):
        ls, ns = eng.prefill([r])
        torch.cuda.synchronize()
        assert rel_err(lb[i], ls[0]) <= 1e-2  # split-K (single) vs full-K (batch) summation order
        assert int(nb[i]) == int(ns[0])


def test_unpack_roundtrip_bit_exact():
    spec = get_spec("gqa-small-64")
    pool = KvPool(spec, n_blocks=64, block_size=64)
    g = torch.Generator(device="cuda").manual_seed(0)
    n1, n2 = 300, 64
    p1 = torch.randn(spec.layers * 2 * spec.kv_heads * n1 * spec.head_dim, generator=g, device="cuda").bfloat16()
    p2 = torch.randn(spec.layers * 2 * spec.kv_heads * n2 * spec.head_dim, generator=g, device="cuda")  # fp32
    b1 = pool.alloc(n1)
    b2 = pool.alloc(n2)
    bt = torch.tensor(list(reversed(b1)) + b2, dtype=torch.int32, device="cuda")
    kv_unpack(pool, [(p1, n1, 0)], bt, elem_width=2)
    kv_unpack(pool, [(p2, n2, len(b1))], bt, elem_width=4)
    torch.cuda.synchronize()
    got1 = pool.gather(list(reversed(b1)), n1).reshape(-1)
    got2 = pool.gather(b2, n2).reshape(-1)
    assert torch.equal(got1, p1)
    assert torch.equal(got2, p2.bfloat16())


def test_graph_replay_matches_eager(setup):
    """CUDA-graph replay (per-shape capture, new metadata copied in) == eager launches."""
    from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
    from paper_2504_11765_b200.store import LookupResult, Outcome
    from paper_2504_11765_b200.codec import KvBlob, make_header

    spec, eng, orc = setup
    prof = spec.profile()
    outs = []
    for rep in range(3):  # capture, then two replays with different content of the same shape
        reqs = []
        for i in range(3):
            pre = combo_tokens([10 * rep + i], [128], spec.vocab)
            kv = eng.generate_doc_kv(pre)
            host = kv.view(torch.uint8).cpu().pin_memory()
            blob = KvBlob.trusted(make_header(prof, [10 * rep + i], len(pre), 0), host)
            reqs.append(PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blob, 0), pre,
                                       query_tokens(rep * 10 + i, 32, spec.vocab)))
        g = prefill_batch(eng, reqs, timed=False, use_graph=True)
        gl = g.logits.clone()
        e = prefill_batch(eng, reqs, timed=False, use_graph=False)
        torch.cuda.synchronize()
        assert rel_err(gl, e.logits) <= 1e-4
        outs.append(gl)
    assert rel_err(outs[1], outs[2]) > 1e-3  # replays really saw new inputs


def test_resident_tier_hit_matches_host_tier_hit():
    """HBM-tier hits (prefix already in pool blocks, nothing loaded) give the same
    logits as host-tier hits (H2D + K3 unpack); a partial last block is copied on
    write, so queries sharing a resident prefix never modify it."""
    from paper_2504_11765_b200.generator import KvGenerator
    from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
    from paper_2504_11765_b200.store import KvKey, LookupResult, Outcome

    spec = get_spec("gqa-small-64")
    per_tok = spec.kv_bytes_per_token()
    eng = Engine(spec, seed=2, pool_tokens=8192, block_size=64, device_cache_bytes=per_tok * 64 * 16)
    gen = KvGenerator(eng, keep_on_device=True)
    prof = spec.profile()
    combos = [((1, 2), (128, 72)), ((3,), (256,))]          # 200 tokens (ragged tail), 256 (block aligned)
    keys, blobs = [], []
    for ids, nt in combos:
        blobs.append(gen.generate(ids, nt))
        keys.append(KvKey(prof.model_hash, ids))
        assert keys[-1] in eng.resident
    before = [eng.pool.gather(eng.resident.acquire(k).blocks, b.header.token_count).clone() for k, b in zip(keys, blobs)]
    for k in keys:
        eng.resident.unpin(k)
    qs = [query_tokens(70 + i, 33, spec.vocab) for i in range(4)]
    # two queries per resident prefix in ONE batch
    idx = [0, 0, 1, 1]
    res = prefill_batch(eng, [PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blobs[j], 0), None, qs[i], keys[j])
                              for i, j in enumerate(idx)], timed=False, use_graph=False)
    host = prefill_batch(eng, [PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blobs[j], 0), None, qs[i], None)
                               for i, j in enumerate(idx)], timed=False, use_graph=False)
    torch.cuda.synchronize()
    assert rel_err(res.logits, host.logits) <= 1e-3
    assert torch.equal(res.next_token, host.next_token)
    for k, b, ref in zip(keys, blobs, before):
        e = eng.resident.acquire(k)
        assert torch.equal(eng.pool.gather(e.blocks, b.header.token_count), ref)
        eng.resident.unpin(k)
    # and against the oracle
    orc = OracleModel(eng.weights)
    toks = gen.tokens(*combos[0])
    _, ref = orc.forward(np.concatenate([toks, qs[0]]))
    _check_logits(res.logits[0], ref, res.next_token[0])


def test_resident_tier_lru_respects_pins():
    spec = get_spec("gqa-small-64")
    per_tok = spec.kv_bytes_per_token()
    eng = Engine(spec, seed=2, pool_tokens=1024, block_size=64, device_cache_bytes=per_tok * 64 * 4)  # 4 blocks
    pay = lambda n: torch.zeros(spec.layers * 2 * spec.kv_heads * n * spec.head_dim, dtype=torch.bfloat16,
                                device="cuda")
    free0 = eng.pool.free_blocks
    assert eng.make_resident("a", pay(128), 128)      # 2 blocks
    assert eng.make_resident("b", pay(100), 100)      # 2 blocks (tier full)
    assert eng.resident.acquire("a") is not None      # pin a (and make it MRU)
    assert eng.make_resident("c", pay(64), 64)        # evicts b (LRU, unpinned)
    assert "b" not in eng.resident and "a" in eng.resident and "c" in eng.resident
    assert not eng.make_resident("d", pay(192), 192)  # 3 blocks: a pinned, cannot fit
    eng.resident.unpin("a")
    assert eng.make_resident("d", pay(192), 192)      # now a and c go
    assert eng.pool.free_blocks == free0 - 3


def test_c2_full_shape_bench_path_matches_oracle():
    """The bench configuration itself (BASELINE configs[1]): Llama-3.2-1B shape at
    full depth, a 5 x 512 composite generated on the GPU and served from the HBM
    tier, 64 query tokens — first-token logits vs the fp32 oracle over the same
    ordered prompt (full-prompt semantics, costs.py:89-99)."""
    from paper_2504_11765_b200.generator import KvGenerator
    from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
    from paper_2504_11765_b200.store import KvKey, LookupResult, Outcome

    spec = get_spec("llama-3.2-1b")
    eng = Engine(spec, seed=0, pool_tokens=4096, device_cache_bytes=spec.kv_bytes_per_token() * 2600)
    gen = KvGenerator(eng, keep_on_device=True)
    docs, ntok = (4211, 17, 905, 3, 77), (512,) * 5
    blob = gen.generate(docs, ntok)
    key = KvKey(spec.profile().model_hash, docs)
    q = query_tokens(12345, 64, spec.vocab)
    r = prefill_batch(eng, [PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blob, 0), None, q, key)], timed=False)
    torch.cuda.synchronize()
    orc = OracleModel(eng.weights)
    kref, ref = orc.forward(np.concatenate([gen.tokens(docs, ntok), q]))
    _check_logits(r.logits[0], ref, r.next_token[0])
    # the cached composite itself (KV written by the QKV epilogue) vs the oracle's KV of the prefix
    got = eng.pool.gather(eng.resident.acquire(key).blocks, 2560).float().cpu()
    eng.resident.unpin(key)
    assert rel_err(got, kref[:, :, :, :2560]) <= TOL


@pytest.mark.parametrize("name,counts", [("tiny", (100, 40, 128)), ("gqa-small-128", (256, 64, 200)),
                                         ("llama-3.2-1b", (512, 512, 512))])
def test_combination_prefix_slices_equal_from_scratch_prefixes(name, counts):
    """SURVEY H-e: one prefill of the ordered combination + slicing gives every prefix
    blob bit-identical (payload, checksum) to generating the prefix from scratch —
    the kernels are row-deterministic in generation mode (no split-K / split-KV)."""
    from paper_2504_11765_b200.generator import KvGenerator

    spec = get_spec(name)
    eng = Engine(spec, seed=5, pool_tokens=4096)
    gen = KvGenerator(eng, keep_on_device=False)
    ids = (31, 7, 19)[: len(counts)]
    factory = gen.for_combination(ids, counts)
    for j in range(1, len(ids) + 1):
        a = factory(ids[:j], counts[:j])()
        b = gen.generate(ids[:j], counts[:j])
        assert a.header == b.header                      # incl. the FNV-1a checksum
        assert torch.equal(a.payload_tensor(), b.payload_tensor())


def test_prepare_uses_one_prefill_per_combination(tmp_path):
    from paper_2504_11765_b200.generator import KvGenerator
    from paper_2504_11765_b200.prefetch import PendingQuery, prepare
    from paper_2504_11765_b200.service import SharedCacheService
    from paper_2504_11765_b200.store import KvKey, KvStore, Outcome

    spec = get_spec("gqa-small-64")
    eng = Engine(spec, seed=5, pool_tokens=4096)
    gen = KvGenerator(eng, keep_on_device=False)
    svc = SharedCacheService(KvStore(tmp_path, 0))
    calls = []
    orig = eng.generate_doc_kv
    eng.generate_doc_kv = lambda toks, *a, **k: (calls.append(len(toks)), orig(toks, *a, **k))[1]
    q = PendingQuery(query_id=1, arrival_time=0.0, k=4, q_tokens=8, doc_ids=(4, 8, 15, 16), doc_tokens=(64, 64, 64, 64))
    q.flagged = True
    prepare(q, None, svc, None, spec.profile(), generator=gen)
    assert calls == [256]                                 # one prefill for the four prefixes
    for j in range(1, 5):
        look = svc.store.get(KvKey(spec.profile().model_hash, q.doc_ids[:j]))
        assert look.outcome is Outcome.DISK_HIT
        ref = gen.generate(q.doc_ids[:j], q.doc_tokens[:j])
        assert look.blob == ref


def test_layer_stream_native_chain_matches_unpack():
    """rdkv_kv_stream_layers (LayerStreamer): per-layer H2D from pinned host memory, the
    unpack of each layer after its copy, one event per layer — the pool ends up exactly as
    a whole-payload kv_unpack of the same bytes leaves it."""
    from paper_2504_11765_b200.engine import LayerStreamer, pack_unpack_jobs

    spec = get_spec("gqa-small-64")
    eng = Engine(spec, seed=0, pool_tokens=4096)
    pool = eng.pool
    g = torch.Generator(device="cuda").manual_seed(1)
    n = 200
    payload = torch.randn(spec.layers * 2 * spec.kv_heads * n * spec.head_dim, generator=g, device="cuda").bfloat16()
    host = payload.view(torch.uint8).cpu().pin_memory()
    blocks_a, blocks_b = pool.alloc(n), pool.alloc(n)
    bt = torch.tensor(blocks_a + blocks_b, dtype=torch.int32, device="cuda")
    kv_unpack(pool, [(payload, n, 0)], bt)  # reference: the device payload, all layers at once
    staging = torch.empty(host.numel(), dtype=torch.uint8, device="cuda")
    jobs = [(staging, n, len(blocks_a))]
    jobs_dev = pack_unpack_jobs(jobs).to("cuda")
    st = LayerStreamer(eng)
    main = torch.cuda.current_stream()
    handles = st.launch(pool, jobs, bt, jobs_dev, main, h2d=[(host, staging)])
    assert all(h for h in handles)
    main.wait_event(st.events[-1])
    torch.cuda.synchronize()
    assert torch.equal(staging, payload.view(torch.uint8))
    assert torch.equal(pool.gather(blocks_b, n), pool.gather(blocks_a, n))


def test_generate_many_pipeline_equals_generate(setup):
    """KvGenerator.generate_many (D2H under the next prefill, checksums left on the device)
    returns blobs byte-identical to generate() of each combination."""
    from paper_2504_11765_b200.generator import KvGenerator

    spec, eng, orc = setup
    gen = KvGenerator(eng, keep_on_device=False)
    combos = [((3, 5), (128, 61)), ((7,), (200,)), ((3, 5, 9), (128, 61, 64))]
    many = gen.generate_many(combos)
    for (ids, counts), b in zip(combos, many):
        ref = gen.generate(ids, counts)
        assert b.header == ref.header
        assert torch.equal(b.payload_tensor(), ref.payload_tensor())
