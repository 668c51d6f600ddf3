"""Pure-Python restatement of the KvStore outcome / byte-LRU law
(TEST INFRASTRUCTURE; see oracle/__init__.py).

Follows store.py:159-172 (insert: cap<=0 or size>cap -> not resident; touch
moves to MRU; evict LRU-first until it fits), :250-280 (memory hit / disk hit /
miss and their counters), :282-289 (contains is side-effect free) and
:299-309 (shrinking capacity evicts).  Same shape as the reference's own test
oracle ReferenceLru (test_store.py:32-59) but tracks the full StoreStats.
"""

from __future__ import annotations


class StoreModel:
    def __init__(self, capacity: int) -> None:
        self.capacity = capacity
        self.lru: list[tuple[tuple, int]] = []   # least recent first
        self.disk: dict[tuple, tuple[int, int]] = {}  # key -> (size, checksum)
        self.stats = dict(memory_hits=0, disk_hits=0, misses=0, evictions=0, corruptions=0,
                          memory_bytes_used=0, memory_capacity_bytes=capacity, disk_bytes_used=0)

    def _resident(self, key):
        return any(k == key for k, _ in self.lru)

    def _touch(self, key, size):
        cap = self.capacity
        if cap <= 0 or size > cap:
            return
        for i, (k, _) in enumerate(self.lru):
            if k == key:
                self.lru.append(self.lru.pop(i))
                return
        while self.lru and self.stats["memory_bytes_used"] + size > cap:
            _, s = self.lru.pop(0)
            self.stats["memory_bytes_used"] -= s
            self.stats["evictions"] += 1
        self.lru.append((key, size))
        self.stats["memory_bytes_used"] += size

    def put(self, key, size, checksum) -> str:
        if key in self.disk or self._resident(key):
            if self.disk[key][1] != checksum:
                return "ImmutableEntryError"
            return "ok"
        self.disk[key] = (size, checksum)
        self.stats["disk_bytes_used"] += size
        self._touch(key, size)
        return "ok"

    def get(self, key) -> tuple[str, int]:
        if self._resident(key):
            self._touch(key, 0)
            self.stats["memory_hits"] += 1
            return "memory_hit", 0
        if key not in self.disk:
            self.stats["misses"] += 1
            return "miss", 0
        size = self.disk[key][0]
        self.stats["disk_hits"] += 1
        self._touch(key, size)
        return "disk_hit", size

    def contains(self, key) -> str:
        if self._resident(key):
            return "in_memory"
        return "on_disk" if key in self.disk else "absent"

    def set_capacity(self, cap: int) -> None:
        self.capacity = cap
        self.stats["memory_capacity_bytes"] = cap
        while self.lru and self.stats["memory_bytes_used"] > cap:
            _, s = self.lru.pop(0)
            self.stats["memory_bytes_used"] -= s
            self.stats["evictions"] += 1

    # Two-phase disk hit, for replaying logs of concurrent runs (SURVEY H-i): the
    # reference decides a disk hit under its lock, reads the file outside it and
    # promotes under the lock again (store.py:250-280), so other operations can
    # interleave between the two halves.
    def read_decision(self, key) -> str:
        """First half of a disk hit: the outcome as decided before the read."""
        if self._resident(key):
            return "memory_hit"
        return "disk_hit" if key in self.disk else "miss"

    def promote(self, key, size) -> None:
        """Second half: count the disk hit and insert into the memory tier."""
        self.stats["disk_hits"] += 1
        self._touch(key, size)


def replay_oplog(oplog, capacity: int) -> dict:
    """Replay a ``KvStore.oplog`` (a real, possibly concurrent run) through the
    store law; asserts every recorded outcome and returns the final stats."""
    m = StoreModel(capacity)
    for op in oplog:
        if op[0] == "put":
            assert m.put(op[1], op[2], op[3]) == op[4], op
        elif op[0] == "read":                      # a disk hit decided; the file is read outside the lock
            assert m.read_decision(op[1]) == "disk_hit", op
        elif op[2] == "disk_hit":                  # ... and promoted once read
            m.promote(op[1], op[3])
        else:
            assert m.get(op[1]) == (op[2], op[3]), op
    return m.stats
