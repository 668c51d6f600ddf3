"""Single-flight semantics of SharedCacheService (reference test_service.py:66-124 scenarios)."""

import threading
import time

import pytest

from paper_2504_11765_b200.codec import ModelProfile, synth_blob
from paper_2504_11765_b200.service import Origin, SharedCacheService
from paper_2504_11765_b200.store import KvStore, Outcome, key_for

P = ModelProfile("tiny", 1, 4, 1, 4, 2)


def test_one_generation_many_waiters(tmp_path):
    svc = SharedCacheService(KvStore(tmp_path, memory_capacity_bytes=0))
    key = key_for(P, [1, 2])
    calls = []
    gate = threading.Event()

    def gen():
        calls.append(1)
        gate.wait(2)
        return synth_blob(P, [1, 2], 3)

    origins = []
    ths = [threading.Thread(target=lambda: origins.append(svc.get_or_generate(key, gen)[1])) for _ in range(8)]
    [t.start() for t in ths]
    time.sleep(0.2)
    gate.set()
    [t.join() for t in ths]
    assert len(calls) == 1
    assert origins.count(Origin.GENERATED) == 1 and origins.count(Origin.WAITED_ON_IN_FLIGHT) == 7
    assert svc.get_or_generate(key, gen)[1] is Origin.DISK_HIT


def test_failure_fans_out_then_retry(tmp_path):
    svc = SharedCacheService(KvStore(tmp_path))
    key = key_for(P, [3])
    gate = threading.Event()

    def bad():
        gate.wait(2)
        raise RuntimeError("generator down")

    errs = []

    def call():
        try:
            svc.get_or_generate(key, bad)
        except RuntimeError as e:
            errs.append(e)

    ths = [threading.Thread(target=call) for _ in range(4)]
    [t.start() for t in ths]
    time.sleep(0.2)
    gate.set()
    [t.join() for t in ths]
    assert len(errs) == 4 and not svc.in_flight(key)
    blob, origin = svc.get_or_generate(key, lambda: synth_blob(P, [3], 2))
    assert origin is Origin.GENERATED


def test_many_keys_one_generation_each(tmp_path):
    svc = SharedCacheService(KvStore(tmp_path, memory_capacity_bytes=1 << 20))
    counts = {}
    lock = threading.Lock()

    def gen_for(ids):
        def g():
            with lock:
                counts[ids] = counts.get(ids, 0) + 1
            time.sleep(0.01)
            return synth_blob(P, ids, 2)
        return g

    def worker(i):
        ids = (i % 4 + 1,)
        svc.get_or_generate(key_for(P, ids), gen_for(ids))

    ths = [threading.Thread(target=worker, args=(i,)) for i in range(64)]
    [t.start() for t in ths]
    [t.join() for t in ths]
    assert counts == {(1,): 1, (2,): 1, (3,): 1, (4,): 1}


def test_memory_hit_origin(tmp_path):
    svc = SharedCacheService(KvStore(tmp_path, memory_capacity_bytes=1 << 20))
    k = key_for(P, [9])
    svc.put(k, synth_blob(P, [9], 2))
    assert svc.get_or_generate(k, lambda: pytest.fail("must not generate"))[1] is Origin.MEMORY_HIT
    assert svc.get(k).outcome is Outcome.MEMORY_HIT
