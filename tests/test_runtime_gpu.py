"""The real-time serving runtime (runtime.py) on a B200: queue-time precompute
on a low-priority stream concurrent with serving, the node control plane,
owner-partitioned generation and NVLink (CUDA IPC) peer fetch with 2 instances
sharing one GPU, and first-token parity of every served query."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _items(n=20, k=3, n_docs=40):
    from paper_2504_11765_b200.workload import zipf_stream

    return zipf_stream(n_docs, 1.0, n, seed=3, k=k, q_tokens=32, doc_tokens=128)


def _expected_tokens(eng, items, k):
    """First token and top-2 margin of every query's full prompt (the miss path)."""
    from paper_2504_11765_b200.engine import QueryRequest
    from paper_2504_11765_b200.model import combo_tokens, query_tokens

    out = {}
    for it in items:
        toks = np.concatenate([combo_tokens(it.doc_ids[:k], it.doc_tokens[:k], eng.spec.vocab),
                               query_tokens(it.query_id, it.q_tokens, eng.spec.vocab)])
        lg, nx = eng.prefill([QueryRequest(toks)])
        top = torch.topk(lg[0].float(), 2).values
        out[it.query_id] = (int(nx[0]), float(top[0] - top[1]))
    return out


def _check_tokens(results, expected):
    for r in results:
        tok, margin = expected[r.query_id]
        assert r.token == tok or margin < 0.05, (r.query_id, r.source, r.token, tok, margin)


def test_single_instance_prefetch_and_reuse():
    from paper_2504_11765_b200.engine import Engine
    from paper_2504_11765_b200.model import get_spec
    from paper_2504_11765_b200.runtime import RuntimeConfig, serve
    from paper_2504_11765_b200.store import KvStore

    spec = get_spec("gqa-small-64")
    k = 3
    items = _items(k=k)
    cfg = RuntimeConfig(k=k, threshold=0.0, max_batch=4, persist="all")
    # throwaway pass on its own engine and store: the first launches of every kernel shape
    # in a fresh process (module load, tensor-map setup) would otherwise delay try 1's
    # generations past try 2's dispatches on a freshly leased box
    with tempfile.TemporaryDirectory() as root:
        warm = Engine(spec, seed=0, pool_tokens=32768, device_cache_bytes=256 << 20)
        serve(warm, KvStore(root, memory_capacity_bytes=0), cfg, items[:8], rate=400.0, tries=1)
        del warm
    eng = Engine(spec, seed=0, pool_tokens=32768, device_cache_bytes=256 << 20)
    expected = _expected_tokens(eng, items, k)
    with tempfile.TemporaryDirectory() as root:
        store = KvStore(root, memory_capacity_bytes=0)
        out = serve(eng, store, cfg, items, rate=400.0, tries=2)
        rep, res = out["summary"], out["results"]
        assert rep["queries"] == 2 * len(items)
        assert sorted(r.index for r in res) == list(range(2 * len(items)))
        assert rep["each_key_generated_once"]
        assert rep["keys_generated"] > 0 and rep["flagged"] > 0
        # try 2 replays the same queries: a combination generated for a query that waited in
        # try 1 is served from HBM (only waiting queries are flagged, prefetch.py:63-72).  Try 2
        # starts as soon as try 1's last query is served, so a generation still in flight then
        # (it keeps running on the low-priority stream; the reference abandons it, sim.py:505-507)
        # can miss try 2's first queries: at least half, and never a wrong source
        made = {ids for qi, ids in out["generated"] if qi < len(items) and len(ids) == k}
        by_id = {it.query_id: tuple(it.doc_ids[:k]) for it in items}
        t2 = [r for r in res if r.index >= len(items) and by_id[r.query_id] in made]
        hits = sum(r.source == "hbm" and r.best == k for r in t2)
        assert t2 and hits >= 0.5 * len(t2), f"{hits} of {len(t2)} try-2 queries served from HBM"
        assert all(r.source in ("hbm", "miss", "peer", "memory", "disk") for r in t2)
        # origin "generated" (served after its own precompute in the same try) depends on timing
        assert rep["origins"].get("generated", 0) + rep["origins"].get("hbm", 0) > 0
        _check_tokens(res, expected)
        # write-behind persistence: every generated prefix is durable and decodes through the store
        store.refresh()
        from paper_2504_11765_b200.store import CacheTier, KvKey

        mh = spec.profile().model_hash
        for it in items:
            for j in range(1, k + 1):
                key = KvKey(mh, it.doc_ids[:j])
                if key in eng.resident:
                    assert store.contains(key) is not CacheTier.ABSENT
        assert rep["qps"] > 0 and rep["latency_ms"]["p99"] >= rep["latency_ms"]["p50"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _two_instance_worker(rank, world, port, root, q):
    import torch.distributed as dist

    from paper_2504_11765_b200.engine import Engine
    from paper_2504_11765_b200.model import get_spec
    from paper_2504_11765_b200.multi import PeerPools
    from paper_2504_11765_b200.runtime import RuntimeConfig, serve
    from paper_2504_11765_b200.store import KvStore

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)  # both instances share the one GPU of this box
        spec = get_spec("gqa-small-64")
        k = 3
        eng = Engine(spec, seed=0, pool_tokens=32768, device_cache_bytes=256 << 20)
        peers = PeerPools(eng)
        items = _items(n=24, k=k)
        expected = _expected_tokens(eng, items, k) if rank == 0 else None
        store = KvStore(root, memory_capacity_bytes=0)
        cfg = RuntimeConfig(k=k, threshold=0.0, max_batch=2, persist="composite")
        out = serve(eng, store, cfg, items, rate=300.0, tries=2, rank=rank, world=world, peers=peers)
        if rank == 0:
            _check_tokens(out["results"], expected)
            rep = out["summary"]
            q.put((rep["each_key_generated_once"], rep["counters"], rep["sources"], rep["queries"],
                   sorted({r.rank for r in out["results"]})))
        peers.close()
    finally:
        dist.destroy_process_group()


def test_two_instances_share_one_gpu_peer_fetch():
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as root:
        port = _free_port()
        ps = [ctx.Process(target=_two_instance_worker, args=(r, world, port, root, q)) for r in range(world)]
        [p.start() for p in ps]
        once, counters, sources, n, ranks = q.get(timeout=240)
        [p.join(timeout=120) for p in ps]
    assert all(p.exitcode == 0 for p in ps)
    assert once and n == 48
    assert ranks == [0, 1]                                      # both instances pulled from the central FIFO
    assert sum(counters["generated_by_rank"]) == counters["keys_generated"] > 0
    assert all(g > 0 for g in counters["generated_by_rank"])    # owner-partitioned: both ranks generated
    assert counters["peer_fetches"] > 0 and sources.get("peer", 0) > 0   # NVLink (IPC) pulls from the peer's HBM


def test_runtime_store_path_oplog_replays():
    """HBM tier off: generated prefixes live only in the shared store (memory tier
    + disk); try 2 is served through KvStore.get.  The real store's operation log
    of the concurrent run (serve thread gets, writer puts) replays into the store
    law with identical outcomes and stats (SURVEY H-i)."""
    from dataclasses import asdict

    from oracle.store_ref import replay_oplog
    from paper_2504_11765_b200.engine import Engine
    from paper_2504_11765_b200.model import get_spec
    from paper_2504_11765_b200.runtime import RuntimeConfig, serve
    from paper_2504_11765_b200.store import KvStore

    spec = get_spec("gqa-small-64")
    k = 3
    eng = Engine(spec, seed=0, pool_tokens=32768, device_cache_bytes=0)
    items = _items(k=k)
    expected = _expected_tokens(eng, items, k)
    cap = 3 << 20  # a few composites: the memory tier evicts
    with tempfile.TemporaryDirectory() as root:
        store = KvStore(root, memory_capacity_bytes=cap)
        store.oplog = []
        out = serve(eng, store, RuntimeConfig(k=k, threshold=0.0, max_batch=4, persist="all"), items,
                    rate=400.0, tries=2)
        rep = out["summary"]
        assert rep["each_key_generated_once"] and rep["queries"] == 2 * len(items)
        assert {"memory", "disk"} & set(rep["sources"])            # served through the store tiers
        _check_tokens(out["results"], expected)
        want = replay_oplog(store.oplog, cap)
        got = asdict(store.stats())
        assert all(got[f] == v for f, v in want.items()), (got, want)
        gets = [op for op in store.oplog if op[0] == "get"]
        assert len(gets) >= len(out["access_log"]) > 0


@pytest.mark.parametrize("disk_gbps,expect_disk", [(1e-6, False), (1e6, True)])
def test_cost_aware_dispatch(disk_gbps, expect_disk):
    """Opt-in cost-aware dispatch: composites that live only on disk are read when the
    predicted read beats recomputing their tokens, else recomputed (DISK_SKIPPED), and
    the first tokens are the same either way."""
    from paper_2504_11765_b200.engine import Engine
    from paper_2504_11765_b200.generator import KvGenerator
    from paper_2504_11765_b200.model import get_spec
    from paper_2504_11765_b200.runtime import RuntimeConfig, serve
    from paper_2504_11765_b200.store import KvKey, KvStore

    spec = get_spec("gqa-small-64")
    k = 3
    eng = Engine(spec, seed=0, pool_tokens=32768, device_cache_bytes=0)
    items = _items(n=12, k=k)
    expected = _expected_tokens(eng, items, k)
    gen = KvGenerator(eng, keep_on_device=False)
    with tempfile.TemporaryDirectory() as root:
        store = KvStore(root, memory_capacity_bytes=0)           # disk only (the paper's shared setting)
        for it in items:
            key = KvKey(spec.profile().model_hash, tuple(it.doc_ids[:k]))
            if store.contains(key).name == "ABSENT":
                store.put(key, gen.generate(it.doc_ids[:k], it.doc_tokens[:k]))
        cfg = RuntimeConfig(k=k, threshold=10.0, prefetch=False, max_batch=4, cost_aware=True,
                            disk_gbps=disk_gbps, prefill_s_per_token=1e-5)
        out = serve(eng, store, cfg, items, rate=200.0, tries=1)
        rep = out["summary"]
        assert rep["queries"] == len(items)
        if expect_disk:
            assert rep["sources"].get("disk", 0) == len(items) and rep["counters"]["disk_skipped"] == 0
        else:
            assert rep["sources"].get("miss", 0) == len(items)
            assert rep["counters"]["disk_skipped"] == len(items)
        _check_tokens(out["results"], expected)


@pytest.mark.parametrize("chunk", [0, 96], ids=["whole-prompts", "chunked-prefill"])
def test_runtime_continuous_batching_decode(chunk):
    """decode_tokens > 0: every query generates more tokens after its first one while new
    queries' prefills join the running batch between decode steps (chunked: prompts enter
    96 tokens per forward, sharing forwards with the decodes).  Each query's tokens equal a
    stand-alone greedy decode of its full prompt where the margins are clear, all pool
    blocks come back, and the summary reports decode throughput / TPOT."""
    from paper_2504_11765_b200 import decode
    from paper_2504_11765_b200.engine import Engine
    from paper_2504_11765_b200.model import combo_tokens, get_spec, query_tokens
    from paper_2504_11765_b200.prefill import PrefillRequest
    from paper_2504_11765_b200.runtime import RuntimeConfig, serve
    from paper_2504_11765_b200.store import KvStore, LookupResult, Outcome

    spec = get_spec("gqa-small-128")
    k, n_dec = 3, 6
    eng = Engine(spec, seed=0, pool_tokens=32768, device_cache_bytes=64 << 20)
    items = _items(n=12, k=k)
    # reference: each full prompt decoded alone (miss path), with the top-2 margin of every step
    ref = {}
    for it in items:
        toks = np.concatenate([combo_tokens(it.doc_ids[:k], it.doc_tokens[:k], spec.vocab),
                               query_tokens(it.query_id, it.q_tokens, spec.vocab)])
        seqs = decode.start(eng, [PrefillRequest(LookupResult(Outcome.MISS), toks[:0], toks)], n_dec + 1)
        margins = []
        try:
            while not seqs[0].done:
                decode.step(eng, seqs)
                top = torch.topk(eng._decode_step.logits[0].float(), 2).values
                margins.append(float(top[0] - top[1]))
            ref[it.query_id] = (list(seqs[0].tokens), margins)
        finally:
            decode.retire(eng, seqs[0])
    free0 = eng.pool.free_blocks
    with tempfile.TemporaryDirectory() as root:
        cfg = RuntimeConfig(k=k, threshold=0.0, max_batch=4, persist="all", decode_tokens=n_dec,
                            prefill_chunk=chunk)
        out = serve(eng, KvStore(root, memory_capacity_bytes=0), cfg, items, rate=400.0, tries=1)
    rep = out["summary"]
    assert rep["queries"] == len(items)
    assert rep["decode"]["queries"] == len(items) and rep["decode"]["tokens"] == len(items) * (n_dec + 1)
    assert rep["decode"]["tpot_ms"]["p50"] > 0 and rep["decode"]["tokens_per_s"] > 0
    compared = 0
    for r in out["results"]:
        assert r.n_tokens == n_dec + 1 and len(r.tokens) == n_dec + 1 and r.done >= r.first_token
        assert r.tokens[0] == r.token
        toks, margins = ref[r.query_id]
        # same greedy continuation until a near-tie step (margin < 0.05) lets bf16 noise pick
        # the other token; the first token is covered by _check_tokens' rule
        if r.token != toks[0]:
            continue
        for j in range(1, n_dec + 1):
            if margins[j - 1] < 0.05:
                break
            assert r.tokens[j] == toks[j], (r.query_id, j, r.tokens, toks)
            compared += 1
    assert compared >= len(items)
    eng.resident.clear()
    assert eng.pool.free_blocks == free0
