"""Host logic of the multi-instance runtime on CPU (no GPU): world-size-2 gloo
processes share one node control plane; rank 0's Driver replays Poisson
arrivals into the central FIFO and flags queries at the threshold
(prefetch.scan), both ranks pull queries and serve their owner-partitioned
generation rings with the cross-process single-flight claims.  Checks every
query is dispatched exactly once and every key generated exactly once, by its
combination's owner."""

import os
import socket
import threading
import time

import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_11765_b200.control import ControlPlane, Counter, QState
from paper_2504_11765_b200.multi import owner_rank
from paper_2504_11765_b200.runtime import STOP, Driver, RuntimeConfig, arrivals_for_try, claim_keys, finish_keys
from paper_2504_11765_b200.store import KvKey
from paper_2504_11765_b200.workload import zipf_stream

MH = 0xC0FFEE


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cp = ControlPlane(name, rank, world, create=rank == 0)
        dist.barrier()
        items = zipf_stream(30, 1.0, 40, seed=7, k=3, q_tokens=8, doc_tokens=16)
        cfg = RuntimeConfig(k=3, threshold=0.002)
        served, generated, owned_ok = [], [], True

        def serve():
            while not cp.counter(STOP):
                got = cp.pop_query()
                if got is None:
                    time.sleep(1e-4)
                    continue
                assert cp.qstate_cas(got[0], QState.QUEUED, QState.DISPATCHED)
                time.sleep(0.004)  # service time: the queue builds, so queries get flagged
                served.append(got[0])
                cp.qstate_cas(got[0], QState.DISPATCHED, QState.DONE)

        def generate():
            nonlocal owned_ok
            while not cp.counter(STOP):
                req = cp.pop_request()
                if req is None:
                    time.sleep(1e-4)
                    continue
                _, ids, counts = req
                owned_ok &= owner_rank(KvKey(MH, tuple(ids)), world) == rank
                keys = [KvKey(MH, tuple(ids[:j])) for j in range(1, len(ids) + 1)]
                won = claim_keys(cp, keys)
                generated.extend(keys[j - 1].doc_ids for j in won)
                finish_keys(cp, [keys[j - 1] for j in won])

        ths = [threading.Thread(target=serve), threading.Thread(target=generate)]
        [t.start() for t in ths]
        flagged = 0
        if rank == 0:
            drv = Driver(cp, cfg, MH)
            for t in range(2):
                drv.run(arrivals_for_try(items, 400.0, 1, t + 1), t * len(items), time.monotonic())
            flagged = drv.flagged
            cp.add(STOP)
        [t.join() for t in ths]
        dist.barrier()
        q.put((rank, served, generated, owned_ok, flagged, cp.counters()))
        dist.barrier()
        cp.close(unlink=rank == 0)
    finally:
        dist.destroy_process_group()


def test_two_rank_runtime_protocol():
    world = 2
    name = f"/rdkv_rtcpu_{os.getpid()}"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    [p.start() for p in ps]
    res = sorted(q.get(timeout=180) for _ in range(world))
    [p.join(timeout=60) for p in ps]
    assert all(p.exitcode == 0 for p in ps)
    served = sorted(i for r in res for i in r[1])
    assert served == list(range(80))                       # 2 tries x 40 queries, each dispatched once
    assert all(len(r[1]) > 0 for r in res)                 # both instances pulled from the central FIFO
    gen = [k for r in res for k in r[2]]
    assert len(gen) == len(set(gen)) > 0                   # each key generated exactly once
    assert all(r[3] for r in res)                          # requests reached the combination's owner
    counters = res[0][5]
    assert counters["keys_generated"] == len(gen) == sum(counters["generated_by_rank"])
    assert res[0][4] > 0                                   # queries were flagged at the threshold
