"""Peer HBM-tier fetch (K3p over CUDA IPC): two instances, one process each.

The driver's GPU box has one GPU, so both ranks share cuda:0 — the IPC mapping
and the gather kernel are the same code that reads a peer GPU over NVLink.
Each rank generates the document KV of the combinations it owns
(owner_rank, multi.py), the resident directory is exchanged over gloo, every
rank pulls the combinations it does not own from the owner's pool, and the
fetched blocks must equal a local recomputation bit for bit (the kernels are
deterministic)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

COMBOS = [((1, 2), (128, 72)), ((5,), (300,)), ((7, 8, 9), (64, 64, 64)), ((11,), (64,)), ((3, 4), (100, 28)),
          ((20,), (1,)), ((21, 22), (256, 256))]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_11765_b200.engine import Engine
        from paper_2504_11765_b200.generator import KvGenerator
        from paper_2504_11765_b200.model import get_spec
        from paper_2504_11765_b200.multi import PeerPools, ResidentDirectory, owner_rank
        from paper_2504_11765_b200.store import KvKey

        torch.cuda.set_device(0)
        spec = get_spec("gqa-small-64")
        eng = Engine(spec, seed=3, pool_tokens=4096, device_cache_bytes=spec.kv_bytes_per_token() * 64 * 64)
        gen = KvGenerator(eng, keep_on_device=True)
        prof = spec.profile()
        keys = [KvKey(prof.model_hash, ids) for ids, _ in COMBOS]
        for (ids, nt), k in zip(COMBOS, keys):
            if owner_rank(k, world) == rank:
                gen.generate(ids, nt)
        dist.barrier()
        peers = PeerPools(eng)
        directory = ResidentDirectory.exchange(eng)
        fetched, exact, holders_ok = 0, [], True
        for (ids, nt), k in zip(COMBOS, keys):
            holders_ok &= directory.holder(k) == owner_rank(k, world)
            if directory.holder(k) != rank:
                assert peers.fetch(directory, k)
                fetched += 1
        torch.cuda.synchronize()
        for (ids, nt), k in zip(COMBOS, keys):
            e = eng.resident.acquire(k)
            got = eng.pool.gather(e.blocks, e.n_tokens).reshape(-1)
            eng.resident.unpin(k)
            ref = eng.generate_doc_kv(gen.tokens(ids, nt))
            torch.cuda.synchronize()
            exact.append(bool(torch.equal(got, ref)))
        dist.barrier()  # holders keep their entries until every rank has fetched
        peers.close()
        q.put((rank, fetched, exact, holders_ok))
    finally:
        dist.destroy_process_group()


def test_two_instances_fetch_peer_resident_kv():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    res = sorted(q.get(timeout=300) for _ in range(world))
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    assert sum(r[1] for r in res) == len(COMBOS)      # every key fetched by exactly the non-owner
    assert all(r[1] > 0 for r in res)                 # both ranks pulled something from the other
    assert all(all(r[2]) for r in res), res           # bit-exact against local recomputation
    assert all(r[3] for r in res)                     # directory agrees with owner_rank
