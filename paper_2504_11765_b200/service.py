"""Shared cache manager: single-flight KV generation over a :class:`KvStore`.

Drop-in for ``ragdcache.service.SharedCacheService`` (reference
service.py:77-140): concurrent requests for one absent key run ``generate()``
exactly once system-wide; late requesters block (outside the lock) until the
owner's blob is durable in the store, and a generator failure is re-raised to
every waiter and clears the in-flight mark so a later call may retry
(service.py:87-127).

On B200 ``generate`` is a :class:`~paper_2504_11765_b200.engine.KvGenerator`
bound to a key: it runs the document prefill on the owning GPU through the
C ABI, which releases the GIL, so waiters on other GPUs' worker threads make
progress meanwhile.  The reference's TCP protocol (service.py:143-414) is out
of scope: one host shares through this in-process manager, the filesystem and
NVLink.
"""

from __future__ import annotations

import threading
from enum import Enum
from typing import Callable

from .codec import KvBlob
from .store import CacheTier, KvKey, KvStore, LookupResult, Outcome


class Origin(Enum):
    MEMORY_HIT = "memory_hit"
    DISK_HIT = "disk_hit"
    GENERATED = "generated"
    WAITED_ON_IN_FLIGHT = "waited_on_in_flight"


class _InFlight:
    """One pending generation: an event plus its outcome."""

    __slots__ = ("done", "blob", "error")

    def __init__(self) -> None:
        self.done = threading.Event()
        self.blob: KvBlob | None = None
        self.error: BaseException | None = None

    def wait(self) -> KvBlob:
        self.done.wait()
        if self.error is not None:
            raise self.error
        assert self.blob is not None
        return self.blob


class SharedCacheService:
    """Thread-safe facade adding request deduplication over a KvStore."""

    _FROM_OUTCOME = {Outcome.MEMORY_HIT: Origin.MEMORY_HIT, Outcome.DISK_HIT: Origin.DISK_HIT}

    def __init__(self, store: KvStore) -> None:
        self.store = store
        self._lock = threading.Lock()
        self._pending: dict[KvKey, _InFlight] = {}

    def get_or_generate(self, key: KvKey, generate: Callable[[], KvBlob]) -> tuple[KvBlob, Origin]:
        """Blob for ``key``, produced at most once; ``generate`` must be
        deterministic for the key."""
        while True:
            found = self.store.get(key)
            if found.outcome is not Outcome.MISS:
                return found.blob, self._FROM_OUTCOME[found.outcome]
            with self._lock:
                slot = self._pending.get(key)
                mine = slot is None
                if mine:
                    if self.store.contains(key) is not CacheTier.ABSENT:
                        continue  # a generation finished between get() and here
                    slot = self._pending[key] = _InFlight()
            if not mine:
                return slot.wait(), Origin.WAITED_ON_IN_FLIGHT
            try:
                blob = generate()
                self.store.put(key, blob)
            except BaseException as exc:
                with self._lock:
                    self._pending.pop(key, None)
                slot.error = exc
                slot.done.set()
                raise
            with self._lock:
                self._pending.pop(key, None)
            slot.blob = blob
            slot.done.set()
            return blob, Origin.GENERATED

    def in_flight(self, key: KvKey) -> bool:
        with self._lock:
            return key in self._pending

    # the service stands in for the store (service.py:129-140)
    def get(self, key: KvKey) -> LookupResult:
        return self.store.get(key)

    def put(self, key: KvKey, blob: KvBlob) -> None:
        self.store.put(key, blob)

    def contains(self, key: KvKey) -> CacheTier:
        return self.store.contains(key)

    def stats(self):
        return self.store.stats()
