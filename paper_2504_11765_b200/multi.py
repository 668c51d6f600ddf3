"""Multi-instance sharding: one model instance per GPU.

Queries are independent units, so N instances serve N disjoint shards of the
query stream with no data-path collective.  Document-KV precompute is
partitioned by a deterministic function of the key,
``owner = int(file_stem, 16) mod N`` (store.py:71-74 gives the stem), so any
instance can ask for any key and exactly one GPU generates it.

Sharing happens through the shared disk tier (every rank's ``KvStore`` points
at the same root; ``KvStore.refresh`` picks up entries other ranks appended to
the manifest) and, for payloads resident in a peer GPU's HBM, through NVLink
(:class:`PeerPools`: CUDA-IPC maps of every rank's paged pool, gathered block by
block).  The *logical* outcome of every access is still decided by the store, so
hit/miss accounting stays bit-exact; placement only changes where the bytes come from.

Control-plane exchange (which keys each rank holds in HBM, :class:`ResidentDirectory`) uses
``torch.distributed`` object collectives — metadata only.
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


class ResidentDirectory:
    """Which rank holds which key in its HBM tier, and in which pool blocks.

    Built by an all-gather of (key, blocks, n_tokens) over a process group
    (gloo or nccl object collective: metadata only).  It is a snapshot: the
    holders must not evict the listed entries until the fetch phase that
    uses it has ended (``PeerPools.fetch`` callers bracket it with barriers)."""

    def __init__(self, holdings: Sequence[Sequence[tuple]]) -> None:
        self.where: dict[KvKey, tuple[int, list[int], int]] = {}
        for r, entries in enumerate(holdings):
            for key, blocks, n in entries:
                self.where.setdefault(key, (r, list(blocks), int(n)))

    @classmethod
    def exchange(cls, engine, group=None) -> "ResidentDirectory":
        import torch.distributed as dist

        torch.cuda.synchronize(engine.device)  # the listed blocks are fully written before anyone reads them
        mine = [((k.model_hash, k.doc_ids), e.blocks, e.n_tokens) for k, e in engine.resident.items()
                if isinstance(k, KvKey)]
        out: list = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, mine, group=group)
        return cls([[(KvKey(m, ids), b, n) for (m, ids), b, n in lst] for lst in out])

    def holder(self, key: KvKey) -> int | None:
        hit = self.where.get(key)
        return hit[0] if hit else None

    def entry(self, key: KvKey):
        return self.where.get(key)


class PeerPools:
    """Every rank's paged KV pool mapped into this process (CUDA IPC), so K3p
    (``rdkv_kv_peer_gather``) can read a peer's HBM-tier blocks over NVLink."""

    def __init__(self, engine, group=None) -> None:
        import ctypes as C

        import torch.distributed as dist

        from . import _lib
        from .engine import _L

        self.engine = engine
        lib = _L()
        pool = engine.pool
        h = (C.c_ubyte * 64)()
        off = C.c_int64()
        _lib.check(lib.rdkv_ipc_handle(C.c_void_p(pool.data.data_ptr()), h, C.byref(off)))
        info = (bytes(h), int(off.value), int(pool.slots))
        world = dist.get_world_size(group)
        me = dist.get_rank(group)
        allinfo: list = [None] * world
        dist.all_gather_object(allinfo, info, group=group)
        self.ptr: dict[int, int] = {}
        self.slots: dict[int, int] = {}
        self._opened: list[int] = []
        for r, (hb, o, slots) in enumerate(allinfo):
            self.slots[r] = slots
            if r == me:
                self.ptr[r] = pool.data.data_ptr()
                continue
            base = C.c_void_p()
            _lib.check(lib.rdkv_ipc_open((C.c_ubyte * 64).from_buffer_copy(hb), C.byref(base)))
            self._opened.append(base.value)
            self.ptr[r] = base.value + o

    def close(self) -> None:
        from .engine import _L

        for b in self._opened:
            _L().rdkv_ipc_close(b)
        self._opened = []

    def gather(self, src_rank: int, src_blocks: Sequence[int], dst_blocks: Sequence[int],
               stream: torch.cuda.Stream | None = None) -> None:
        """K3p: copy blocks from rank ``src_rank``'s pool into this rank's pool."""
        from . import _lib
        from .engine import _L, _stream_ptr

        eng, s = self.engine, self.engine.spec
        dev = eng.device
        sb = torch.tensor(list(src_blocks), dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
        db = torch.tensor(list(dst_blocks), dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        _lib.check(_L().rdkv_kv_peer_gather(self.ptr[src_rank], self.slots[src_rank], sb.data_ptr(),
                                            eng.pool.data.data_ptr(), eng.pool.slots, db.data_ptr(), len(db),
                                            s.layers, s.kv_heads, s.head_dim, eng.pool.block_size,
                                            _stream_ptr(st)))
        sb.record_stream(st)
        db.record_stream(st)

    def fetch(self, directory: ResidentDirectory, key: KvKey, stream: torch.cuda.Stream | None = None) -> bool:
        """Place ``key`` in this rank's HBM tier from the peer that holds it
        (False if no peer holds it or it does not fit).  The store still
        decides the logical outcome of the access; this only moves bytes."""
        hit = directory.entry(key)
        if hit is None:
            return False
        rank, src_blocks, n = hit
        eng = self.engine
        if key in eng.resident:
            return True
        dst = eng.resident.reserve(n)
        if dst is None:
            return False
        self.gather(rank, src_blocks, dst, stream)
        eng.resident.commit(key, dst, n)
        return True


class TpGroup:
    """Tensor-parallel group for one instance spread over ``size`` GPUs (C5):
    allocates this rank's zeroed communicator buffer, exchanges CUDA-IPC
    handles over ``group`` (metadata only), maps every peer's buffer and makes
    ``engine``'s model all-reduce its row-parallel projections over them: the
    O / down GEMMs push their bf16 tiles into every rank's receive slot from
    the epilogue (NVLink P2P stores), then rdkv_tp_reduce_resid sums the local
    slots with the residual.  ``engine`` must hold this rank's shard
    (model.shard_weights)."""

    def __init__(self, engine, max_tokens: int, group=None) -> None:
        import ctypes as C

        import torch.distributed as dist

        from . import _lib
        from .engine import _L

        lib = _L()
        self.engine = engine
        self.group = group
        self.rank, self.size = dist.get_rank(group), dist.get_world_size(group)
        engine.tp_rank = self.rank  # its KV heads of full-model blobs: [rank * kv_heads, (rank + 1) * kv_heads)
        self.max_elems = max_tokens * engine.spec.hidden
        nbytes = int(lib.rdkv_tp_comm_bytes(self.max_elems, self.size))
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=engine.device)
        torch.cuda.synchronize(engine.device)
        h = (C.c_ubyte * 64)()
        off = C.c_int64()
        _lib.check(lib.rdkv_ipc_handle(C.c_void_p(self.buf.data_ptr()), h, C.byref(off)))
        allinfo: list = [None] * self.size
        dist.all_gather_object(allinfo, (bytes(h), int(off.value)), group=group)
        bases = (C.c_void_p * self.size)()
        self._opened = []
        for r, (hb, o) in enumerate(allinfo):
            if r == self.rank:
                bases[r] = self.buf.data_ptr()
                continue
            base = C.c_void_p()
            _lib.check(lib.rdkv_ipc_open((C.c_ubyte * 64).from_buffer_copy(hb), C.byref(base)))
            self._opened.append(base.value)
            bases[r] = base.value + o
        comm = C.c_void_p()
        _lib.check(lib.rdkv_tp_comm_create(self.rank, self.size, bases, self.max_elems, C.byref(comm)))
        self.comm = comm
        _lib.check(lib.rdkv_model_set_tp(engine.model._h, comm))
        dist.barrier(group=group)

    def push(self, partial: torch.Tensor, buf: int = 0, stream=None) -> None:
        """Store this rank's dense [rows, cols] bf16 partial into its slot of parity
        ``buf`` in every rank's buffer (what the PUSH GEMM epilogue does in-kernel)."""
        from . import _lib
        from .engine import _L, _stream_ptr

        rows, cols = partial.shape
        _lib.check(_L().rdkv_tp_push(self.comm, partial.data_ptr(), rows, cols, buf, _stream_ptr(stream)))

    def reduce_resid(self, x: torch.Tensor, buf: int = 0, stream=None) -> None:
        """x[rows, cols] += sum of the partials every rank pushed in parity ``buf``."""
        from . import _lib
        from .engine import _L, _stream_ptr

        rows, cols = x.shape
        _lib.check(_L().rdkv_tp_reduce_resid(self.comm, x.data_ptr(), x.stride(0), rows, cols, buf,
                                             _stream_ptr(stream)))

    def gather_payload(self, local: torch.Tensor, n_tokens: int, root: int = 0) -> torch.Tensor | None:
        """Assemble the full-model payload [L][2][Hkv][n][dh] from every rank's share
        [L][2][Hkv/T][n][dh] (document prefill on a TP instance) into HBM on ``root``:
        each rank writes its heads with one strided copy straight into the root's
        gather buffer over NVLink (CUDA-IPC mapping), then the group synchronises.
        Returns the full payload (bf16, flat) on ``root``, None elsewhere."""
        import ctypes as C

        import torch.distributed as dist

        from . import _lib
        from .engine import _L

        s = self.engine.spec
        group = self.group
        # ``root`` is a rank of this TP group; collectives address it by its global rank
        root_global = dist.get_global_rank(group, root) if group is not None else root
        part = s.layers * 2 * s.kv_heads * n_tokens * s.head_dim  # elements of one rank's share
        full = part * self.size
        if not hasattr(self, "_gather") or self._gather_elems < full:
            # (re)size the root's gather buffer and (re)map it everywhere
            if hasattr(self, "_gather") and self._gather_peer:
                _L().rdkv_ipc_close(self._gather_peer)
            info = [None]
            if self.rank == root:
                self._gather_buf = torch.empty(full, dtype=torch.bfloat16, device=self.engine.device)
                h = (C.c_ubyte * 64)()
                off = C.c_int64()
                _lib.check(_L().rdkv_ipc_handle(C.c_void_p(self._gather_buf.data_ptr()), h, C.byref(off)))
                info = [(bytes(h), int(off.value))]
            dist.broadcast_object_list(info, src=root_global, group=group)
            self._gather_peer = None
            if self.rank == root:
                self._gather = self._gather_buf.data_ptr()
            else:
                base = C.c_void_p()
                _lib.check(_L().rdkv_ipc_open((C.c_ubyte * 64).from_buffer_copy(info[0][0]), C.byref(base)))
                self._gather_peer = base.value
                self._gather = base.value + info[0][1]
            self._gather_elems = full
        # the root may still be hashing / copying the previous payload out of the gather
        # buffer: nobody writes into it before the root has arrived here
        torch.cuda.current_stream(self.engine.device).synchronize()
        dist.barrier(group=group)
        width = s.kv_heads * n_tokens * s.head_dim * 2          # bytes of this rank's heads per (layer, K|V)
        pitch = width * self.size                               # bytes of all heads per (layer, K|V)
        dst = self._gather + self.rank * width
        st = torch.cuda.current_stream(self.engine.device)
        _lib.check(_L().rdkv_memcpy_2d(dst, pitch, local.data_ptr(), width, width, s.layers * 2, st.cuda_stream))
        st.synchronize()
        dist.barrier(group=group)
        return self._gather_buf[:full] if self.rank == root else None

    def generate_blob(self, tokens, doc_ids, root: int = 0):
        """Document-KV generation on a TP instance (the ``generate()`` plugin body for
        C5): every rank prefills the combination for its KV heads, the shares are
        gathered over NVLink on ``root``, hashed there on the GPU and copied once
        into pinned host memory.  Returns the full-model ``KvBlob`` on ``root``."""
        from dataclasses import replace

        import numpy as np

        from .codec import KvBlob, fnv1a64_device, make_header

        eng = self.engine
        n = len(tokens)
        local = eng.generate_doc_kv(np.asarray(tokens, np.int32))
        full = self.gather_payload(local, n, root)
        if self.rank != root:
            return None
        s = eng.spec
        full_spec = replace(s, n_heads=s.n_heads * self.size, kv_heads=s.kv_heads * self.size, ffn=s.ffn * self.size)
        raw = full.view(torch.uint8)
        checksum = fnv1a64_device(raw)
        host = torch.empty(raw.numel(), dtype=torch.uint8, pin_memory=True)
        host.copy_(raw)
        return KvBlob.trusted(make_header(full_spec.profile(), tuple(doc_ids), n, checksum), host)

    def close(self) -> None:
        from .engine import _L

        if getattr(self, "_gather_peer", None):
            _L().rdkv_ipc_close(self._gather_peer)
            self._gather_peer = None
        if self.comm:
            _L().rdkv_model_set_tp(self.engine.model._h, None)
            _L().rdkv_tp_comm_destroy(self.comm)
            self.comm = None
        for b in self._opened:
            _L().rdkv_ipc_close(b)
        self._opened = []
