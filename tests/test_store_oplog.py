"""SURVEY H-i: a concurrent run's store operation log, replayed into the store
law restated in oracle/store_ref.StoreModel (pinned to the reference's own
op-log golden in test_oracle.py), reproduces every outcome and the final
StoreStats.  Several threads put and get at once, as the runtime's serving,
generation and writer threads do."""

import random
import threading
from dataclasses import asdict

from oracle.store_ref import replay_oplog
from paper_2504_11765_b200.codec import ModelProfile, synth_blob
from paper_2504_11765_b200.store import KvKey, KvStore

P = ModelProfile("oplog", 1, 8, 2, 4, 2)


replay = replay_oplog


def test_concurrent_oplog_replays_into_the_store_law(tmp_path):
    cap = 6 * (16 + 8 + 30 + 2 * 1 * 2 * 4 * 24 * 2)  # about six 1-doc blobs of 24 tokens
    store = KvStore(tmp_path, memory_capacity_bytes=cap)
    store.oplog = []
    keys = [KvKey(P.model_hash, (i,)) for i in range(24)]
    blobs = {k: synth_blob(P, k.doc_ids, 24 + (k.doc_ids[0] % 3) * 8) for k in keys}

    def writer(part):
        for k in part:
            store.put(k, blobs[k])

    def reader(seed):
        rng = random.Random(seed)
        for _ in range(300):
            store.get(keys[rng.randrange(len(keys))])

    ths = [threading.Thread(target=writer, args=(keys[i::3],)) for i in range(3)]
    ths += [threading.Thread(target=reader, args=(s,)) for s in range(4)]
    [t.start() for t in ths]
    [t.join() for t in ths]
    # a deterministic tail after the concurrent phase so every outcome is exercised whatever the
    # interleaving was (readers can finish before the writers reach most keys): the oldest keys
    # were evicted from the memory tier (disk hits), the newest are resident, one key is absent
    store.put(keys[0], blobs[keys[0]])
    for k in keys:
        store.get(k)
    store.get(KvKey(P.model_hash, (999,)))
    got = asdict(store.stats())
    want = replay(store.oplog, cap)
    for f, v in want.items():
        assert got[f] == v, (f, got[f], v)
    outcomes = {op[2] for op in store.oplog if op[0] == "get"}
    assert outcomes == {"memory_hit", "disk_hit", "miss"}   # every branch exercised
