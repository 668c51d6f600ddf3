"""Multi-instance host logic on CPU: world_size-2 gloo processes (no GPU).

Checks owner-partitioned precompute over a shared disk root, query sharding,
and that every rank ends up seeing every
key through the shared store (KvStore.refresh)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_11765_b200.codec import ModelProfile, synth_blob
from paper_2504_11765_b200.multi import owned, owner_rank, shard
from paper_2504_11765_b200.service import Origin, SharedCacheService
from paper_2504_11765_b200.store import KvKey, KvStore, Outcome
from paper_2504_11765_b200.workload import zipf_stream

P = ModelProfile("tiny", 1, 4, 1, 4, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, root, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        items = zipf_stream(30, 1.0, 40, seed=5, k=2, q_tokens=8, doc_tokens=4)
        mine = shard(items, rank, world)
        keys = sorted({KvKey(P.model_hash, it.doc_ids[:j]) for it in items for j in (1, 2)},
                      key=lambda k: k.doc_ids)
        store = KvStore(root, memory_capacity_bytes=0)
        svc = SharedCacheService(store)
        gen_here = owned(keys, rank, world)
        for k in gen_here:
            _, origin = svc.get_or_generate(k, lambda k=k: synth_blob(P, k.doc_ids, 4 * len(k.doc_ids)))
            assert origin is Origin.GENERATED
        dist.barrier()
        store.refresh()
        seen = sum(store.get(k).outcome is Outcome.DISK_HIT for k in keys)
        agree = all(owner_rank(k, world) == rank for k in gen_here)
        q.put((rank, len(mine), [it.query_id for it in mine], len(gen_here), seen, len(keys), agree))
    finally:
        dist.destroy_process_group()


def test_two_rank_owner_partitioned_precompute(tmp_path):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path), q)) for r in range(world)]
    [p.start() for p in procs]
    res = sorted(q.get(timeout=120) for _ in range(world))
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    ids = sorted(i for r in res for i in r[2])
    assert ids == list(range(40))                       # shards partition the stream
    n_keys = res[0][5]
    assert sum(r[3] for r in res) == n_keys             # each key generated exactly once
    assert all(r[4] == n_keys for r in res)             # every rank sees every key via the shared root
    assert all(r[6] for r in res)                       # each rank generated only keys it owns


def test_owner_rank_deterministic():
    k = KvKey(P.model_hash, (3, 1, 4))
    assert owner_rank(k, 8) == int(k.file_stem, 16) % 8
    assert {owner_rank(KvKey(P.model_hash, (i,)), 4) for i in range(64)} == {0, 1, 2, 3}
    with pytest.raises(ValueError):
        shard([1, 2], 2, 2)
