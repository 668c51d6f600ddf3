"""Multi-instance sharding: one model instance per GPU.

Queries are independent units, so N instances serve N disjoint shards of the
query stream with no data-path collective.  Document-KV precompute is
partitioned by a deterministic function of the key,
``owner = int(file_stem, 16) mod N`` (store.py:71-74 gives the stem), so any
instance can ask for any key and exactly one GPU generates it.

Sharing happens through the shared disk tier (every rank's ``KvStore`` points
at the same root; ``KvStore.refresh`` picks up entries other ranks appended to
the manifest) and, for payloads resident in a peer GPU's HBM, through NVLink
peer copies (:func:`peer_fetch`).  The *logical* outcome of every access is
still decided by the store, so hit/miss accounting stays bit-exact; placement
only changes where the bytes come from.

Control-plane exchange (which keys each rank holds in HBM) uses
``torch.distributed`` object collectives over gloo — metadata only.
"""

from __future__ import annotations

from typing import Sequence

import torch

from .store import KvKey


def owner_rank(key: KvKey, world: int) -> int:
    """Rank that generates ``key`` under owner-partitioned precompute."""
    if world < 1:
        raise ValueError("world must be >= 1")
    return int(key.file_stem, 16) % world


def shard(items: Sequence, rank: int, world: int) -> list:
    """This rank's share of a query stream (round-robin, order preserved)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(items[rank::world])


def owned(keys: Sequence[KvKey], rank: int, world: int) -> list[KvKey]:
    return [k for k in keys if owner_rank(k, world) == rank]


class PeerDirectory:
    """Which rank holds which key in HBM (built by an all-gather of key lists)."""

    def __init__(self, holdings: Sequence[Sequence[KvKey]]) -> None:
        self.where: dict[KvKey, int] = {}
        for r, keys in enumerate(holdings):
            for k in keys:
                self.where.setdefault(k, r)

    @classmethod
    def exchange(cls, my_keys: Sequence[KvKey], group=None) -> "PeerDirectory":
        import torch.distributed as dist

        world = dist.get_world_size(group)
        out: list = [None] * world
        payload = [(k.model_hash, k.doc_ids) for k in my_keys]
        dist.all_gather_object(out, payload, group=group)
        return cls([[KvKey(m, ids) for m, ids in lst] for lst in out])

    def holder(self, key: KvKey) -> int | None:
        return self.where.get(key)


def peer_fetch(src: torch.Tensor, device: torch.device, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Copy a payload resident on a peer GPU into ``device``'s HBM over NVLink
    (cudaMemcpyPeerAsync under the hood when peer access is enabled)."""
    dst = torch.empty_like(src, device=device)
    if stream is None:
        dst.copy_(src, non_blocking=True)
    else:
        with torch.cuda.stream(stream):
            dst.copy_(src, non_blocking=True)
    return dst
