"""Node control plane (csrc/shm.cpp via control.ControlPlane) on CPU: the
cross-process single-flight law, the residency pin/retract protocol and the
MPMC rings, exercised by several processes at once."""

import multiprocessing as mp
import os
import uuid

import pytest

from paper_2504_11765_b200.control import ControlPlane, Counter, KeyState, QState
from paper_2504_11765_b200.store import KvKey

MH = 0x1234ABCD


def _name():
    return f"/rdkv_test_{os.getpid()}_{uuid.uuid4().hex[:8]}"


def test_single_process_protocol():
    name = _name()
    cp = ControlPlane(name, 0, 2, create=True, table_slots=64, max_blocks=8, ring_slots=4, max_queries=16)
    try:
        k = KvKey(MH, (1, 2, 3))
        assert cp.key_state(k) == (KeyState.ABSENT, -1)
        assert cp.key_cas(k, KeyState.ABSENT, KeyState.GENERATING)
        assert not cp.key_cas(k, KeyState.ABSENT, KeyState.GENERATING)      # single flight
        assert cp.key_state(k) == (KeyState.GENERATING, 0)
        assert cp.key_cas(k, KeyState.GENERATING, KeyState.READY)
        # residency: publish, pin blocks retract, unpin, retract
        assert cp.holder(k) is None and cp.pin(k) is None
        assert cp.publish(k, [5, 6, 7], 150)
        other = ControlPlane(name, 1, 2, create=False)
        assert not other.publish(k, [1], 10)                                 # one holder per key
        assert other.pin(k) == (0, [5, 6, 7], 150)
        assert not cp.retract(k)                                             # a reader holds a pin
        other.unpin(k)
        assert cp.retract(k)
        assert cp.holder(k) is None and other.pin(k) is None
        assert other.publish(k, [1], 10) and cp.holder(k) == 1
        with pytest.raises(Exception):
            ControlPlane._pack_combo([1] * 40, [1] * 40)
        # rings: FIFO order, full / empty
        for i in range(4):
            assert cp.push_query(i, 100 + i, 0.5 * i, 16, (i, i + 1), (8, 8))
        assert not cp.push_query(9, 0, 0.0, 1, (1,), (1,))                   # 4 slots: full
        got = [other.pop_query() for _ in range(4)]
        assert [g[0] for g in got] == [0, 1, 2, 3] and got[2] == (2, 102, 1.0, 16, (2, 3), (8, 8))
        assert other.pop_query() is None
        assert cp.push_request(1, (4, 5), (7, 9), 3)
        assert other.pop_request() == (3, (4, 5), (7, 9)) and other.pop_request() is None
        assert cp.pop_request() is None
        assert cp.qstate_cas(3, QState.NONE, QState.QUEUED) and not cp.qstate_cas(3, QState.NONE, QState.QUEUED)
        assert other.qstate(3) is QState.QUEUED
        assert cp.add(Counter.KEYS_GENERATED, 2) == 2 and other.counter(Counter.KEYS_GENERATED) == 2
        other.close()
    finally:
        cp.close(unlink=True)


def _contender(name, rank, world, n_keys, n_items, q):
    cp = ControlPlane(name, rank, world, create=False)
    won = 0
    for i in range(n_keys):
        if cp.key_cas(KvKey(MH, (i,)), KeyState.ABSENT, KeyState.GENERATING):
            won += 1
            cp.add(Counter.PER_RANK_GENERATED + rank)
    popped = []
    while len(popped) < n_items:
        r = cp.pop_query()
        if r is None:
            if cp.counter(Counter.STORE_PUTS) == 1 and cp.ring_size(0) == 0:
                break
            continue
        popped.append(r[0])
    q.put((rank, won, popped))
    cp.close()


def test_multiprocess_claims_and_mpmc_ring():
    name = _name()
    world, n_keys, n_items = 4, 500, 2000
    cp = ControlPlane(name, 0, world, create=True, table_slots=1024, ring_slots=256, max_queries=16)
    try:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        ps = [ctx.Process(target=_contender, args=(name, r, world, n_keys, n_items, q)) for r in range(world)]
        [p.start() for p in ps]
        for i in range(n_items):
            while not cp.push_query(i, i, 0.0, 1, (i,), (1,)):
                pass
        cp.add(Counter.STORE_PUTS)  # producer done
        res = [q.get(timeout=120) for _ in range(world)]
        [p.join(timeout=60) for p in ps]
        assert all(p.exitcode == 0 for p in ps)
        assert sum(r[1] for r in res) == n_keys                              # each key claimed exactly once
        assert cp.counters()["generated_by_rank"] == [dict((r[0], r[1]) for r in res)[i] for i in range(world)]
        popped = sorted(i for r in res for i in r[2])
        assert popped == list(range(n_items))                                # every record exactly once
    finally:
        cp.close(unlink=True)
