"""Workload streams and prefetch planning vs reference goldens."""

import json
from pathlib import Path

import pytest

from paper_2504_11765_b200.codec import ModelProfile, synth_blob
from paper_2504_11765_b200.costs import cached_prefill_work, prefill_work
from paper_2504_11765_b200.prefetch import PendingQuery, PrefetchState, plan_tasks, prepare, promote, scan
from paper_2504_11765_b200.service import SharedCacheService
from paper_2504_11765_b200.store import CacheTier, KvKey, KvStore
from paper_2504_11765_b200.workload import poissonize, uniform_arrivals, zipf_stream

G = Path(__file__).resolve().parent / "golden"
W = json.loads((G / "workload_golden.json").read_text())
CP = json.loads((G / "costs_prefetch_golden.json").read_text())


@pytest.mark.parametrize("name", [n for n in W if n.startswith("zipf")])
def test_zipf_stream_matches_reference(name):
    _, n, s, q, seed, k = name.split("_")
    items = zipf_stream(int(n), float(s), int(q), seed=int(seed), k=int(k), q_tokens=64, doc_tokens=512)
    assert [list(it.doc_ids) for it in items] == W[name]


def test_arrivals():
    items = zipf_stream(50, 1.0, 20, seed=3)
    assert [t for t, _ in poissonize(items, 40.0, seed=9)] == W["poisson_40_seed9"]
    assert [t for t, _ in uniform_arrivals(items, 100.0)] == W["uniform_100"]


def test_cost_kats():
    for L, D, n, w in CP["prefill_work"]:
        assert prefill_work(L, D, n) == w
    for L, D, q, c, w in CP["cached_prefill_work"]:
        assert cached_prefill_work(L, D, q, c) == w
    assert prefill_work(24, 2048, 128) == 805_306_368  # reference test_costs.py:27


def test_plan_tasks_match_reference(tmp_path):
    prof = ModelProfile("tiny", 1, 4, 1, 4, 2)
    svc = SharedCacheService(KvStore(tmp_path, memory_capacity_bytes=0))
    svc.put(KvKey(prof.model_hash, (4,)), synth_blob(prof, [4], 10))
    for case in CP["plan_tasks"]:
        ids, toks = tuple(case["doc_ids"]), tuple(case["doc_tokens"])
        pq = PendingQuery(0, 0.0, len(ids), 8, doc_ids=ids, doc_tokens=toks)
        got = [[list(t.key.doc_ids), t.est_work] for t in plan_tasks(pq, prof, svc, None)]
        assert got == case["tasks"]


def test_scan_rules():
    q = [PendingQuery(i, float(i), 1, 8, doc_ids=(1,), doc_tokens=(4,)) for i in range(4)]
    assert scan(q, 10.0, 0.0) == [0, 1, 2, 3]
    assert scan(q, 10.0, 0.0) == []
    q2 = [PendingQuery(0, 9.5, 1, 8, doc_ids=(1,)), PendingQuery(1, 8.0, 1, 8, doc_ids=(1,))]
    assert scan(q2, 10.0, 2.0) == [1]


def test_prepare_generates_every_missing_prefix(tmp_path):
    prof = ModelProfile("tiny", 1, 4, 1, 4, 2)
    svc = SharedCacheService(KvStore(tmp_path, memory_capacity_bytes=0))
    made = []

    def gen(ids, counts):
        def g():
            made.append(ids)
            return synth_blob(prof, ids, sum(counts))
        return g

    q = PendingQuery(7, 0.0, 3, 8, doc_ids=(5, 1, 9), doc_tokens=(3, 4, 5), flagged=True)
    prepare(q, None, svc, None, prof, generator=gen)
    assert q.prefetch_state is PrefetchState.READY
    assert made == [(5,), (5, 1), (5, 1, 9)]
    for j in range(1, 4):
        assert svc.contains(KvKey(prof.model_hash, (5, 1, 9)[:j])) is CacheTier.ON_DISK
    q2 = PendingQuery(8, 0.0, 3, 8, doc_ids=(5, 1, 2), doc_tokens=(3, 4, 5), flagged=True)
    prepare(q2, None, svc, None, prof, generator=gen)
    assert made[3:] == [(5, 1, 2)]  # shared prefixes are not regenerated


def test_prepare_failure_resets_state(tmp_path):
    prof = ModelProfile("tiny", 1, 4, 1, 4, 2)
    svc = SharedCacheService(KvStore(tmp_path))

    def boom(ids, counts):
        def g():
            raise RuntimeError("gpu lost")
        return g

    q = PendingQuery(1, 0.0, 1, 8, doc_ids=(2,), doc_tokens=(4,), flagged=True)
    prepare(q, None, svc, None, prof, generator=boom)
    assert q.prefetch_state is PrefetchState.NONE


def test_promote_moves_the_longest_disk_prefix_into_memory(tmp_path):
    prof = ModelProfile("tiny", 2, 256, 4, 64, 2)
    store = KvStore(tmp_path, 0)  # memory tier off while writing: entries land on disk only
    for ids in ((1,), (1, 2)):
        store.put(KvKey(prof.model_hash, ids), synth_blob(prof, ids, 8 * len(ids)))
    q = PendingQuery(7, 0.0, 3, 16, doc_ids=(1, 2, 3), doc_tokens=(8, 8, 8))
    assert promote(q, store, prof) is None  # memory tier off: nothing to do
    store.set_memory_capacity(1 << 20)
    key = promote(q, store, prof)
    assert key == KvKey(prof.model_hash, (1, 2))
    assert store.contains(key) is CacheTier.IN_MEMORY
    assert store.contains(KvKey(prof.model_hash, (1,))) is CacheTier.ON_DISK
    assert store.stats().disk_hits == 1
    assert promote(q, store, prof) is None  # the longest cached prefix is resident now
    assert store.get(key).outcome.name == "MEMORY_HIT"
    assert promote(PendingQuery(8, 0.0, 1, 16, doc_ids=(9,), doc_tokens=(8,)), store, prof) is None
