"""One model instance on one B200: document-KV generation, KV load into a
paged HBM pool, and batched query prefill over cached document prefixes.

This is the device half of the reference path.  Each method names the
reference function whose *semantics* it implements:

* :meth:`Engine.generate_doc_kv` — the payload of ``synth_blob``
  (codec.py:188-224): KV of an ordered document combination computed from
  scratch over its concatenated tokens at positions 0..n-1 (prefetch.py:6-8),
  written by the QKV-GEMM epilogue straight into the `.rdkv` payload layout.
* :meth:`Engine.load_cached` — ``KvStore.get`` payload -> HBM
  (store.py:250-280, ``load_time`` costs.py:102-108): async H2D of the pinned
  payload on a side stream, then the K3 unpack kernel into pool blocks.
* :meth:`Engine.prefill` — ``ttft`` / ``cached_prefill_work``
  (costs.py:89-144): new tokens (uncached documents, then the query) attend
  over the cached prefix plus themselves; the last row yields the first-token
  logits and argmax.

All GPU work goes through librdkv's C ABI; there is no PyTorch compute path.
"""

from __future__ import annotations

import contextlib
import os
import ctypes as C
import threading
from collections import OrderedDict, deque
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .model import ModelSpec, ModelWeights, init_weights


class RdkvModelDesc(C.Structure):
    _fields_ = [("layers", C.c_int32), ("hidden", C.c_int32), ("n_heads", C.c_int32), ("kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32), ("max_pos", C.c_int32),
                ("rope_theta", C.c_float), ("norm_eps", C.c_float), ("flags", C.c_int32)]

RDKV_MODEL_NORM_FOLDED = 1


class RdkvBatch(C.Structure):
    _fields_ = [("n_seqs", C.c_int32), ("n_tokens", C.c_int32), ("max_new", C.c_int32), ("block_size", C.c_int32),
                ("bt_stride", C.c_int32), ("want_logits", C.c_int32),
                ("tokens", C.c_void_p), ("pos", C.c_void_p), ("slot", C.c_void_p), ("seq_start", C.c_void_p),
                ("seq_new", C.c_void_p), ("seq_cached", C.c_void_p), ("block_table", C.c_void_p),
                ("last_row", C.c_void_p), ("kv_base", C.c_void_p), ("kv_slots", C.c_int64),
                ("logits", C.c_void_p), ("next_token", C.c_void_p), ("max_ctx", C.c_int32),
                ("layer_ready", C.c_void_p), ("flags", C.c_int32)]


class RdkvUnpackJob(C.Structure):
    _fields_ = [("src", C.c_void_p), ("n_tokens", C.c_int32), ("first_block", C.c_int32), ("reserved", C.c_int64)]


_UNPACK_DTYPE = np.dtype([("src", "<u8"), ("n_tokens", "<i4"), ("first_block", "<i4"), ("reserved", "<i8")])

_N_SIG = {
    "rdkv_model_create": (C.c_int, [C.POINTER(RdkvModelDesc), C.POINTER(C.c_void_p), C.c_size_t,
                                    C.POINTER(C.c_void_p)]),
    "rdkv_model_destroy": (None, [C.c_void_p]),
    "rdkv_workspace_bytes": (C.c_size_t, [C.c_void_p, C.c_int, C.c_int]),
    "rdkv_forward": (C.c_int, [C.c_void_p, C.POINTER(RdkvBatch), C.c_void_p, C.c_size_t, C.c_void_p]),
    "rdkv_kv_unpack": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                 C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    "rdkv_kv_unpack_heads": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                       C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_void_p]),
    "rdkv_kv_copy_block": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_void_p]),
    "rdkv_kv_stream_layers": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                        C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_int,
                                        C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "rdkv_ipc_handle": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    "rdkv_ipc_open": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "rdkv_ipc_close": (C.c_int, [C.c_void_p]),
    "rdkv_memcpy_2d": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p]),
    "rdkv_kv_peer_gather": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    "rdkv_tp_comm_bytes": (C.c_size_t, [C.c_size_t, C.c_int]),
    "rdkv_tp_comm_create": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "rdkv_tp_comm_destroy": (None, [C.c_void_p]),
    "rdkv_tp_push": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    "rdkv_tp_reduce_resid": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p]),
    "rdkv_model_set_tp": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rdkv_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "rdkv_profile_collect": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_double)]),
}

PROF_CLASSES = ("gemm_qkv", "attention", "norm_embed", "lm_head", "gemm_o", "gemm_gate_up", "gemm_down")


def _L():
    lib = _lib.lib()
    if not getattr(lib, "_engine_sigs", False):
        for name, (res, args) in _N_SIG.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        lib._engine_sigs = True
    return lib


def _nullctx():
    return contextlib.nullcontext()


def _stream_ptr(stream: torch.cuda.Stream | None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


# ----------------------------------------------------------------- KV pool


class KvPool:
    """Paged KV pool in HBM: planes [L][2][Hkv][slots][dh] bf16, slots = n_blocks * block_size.

    Head-major like the blob payload, so unpacking a blob block is one
    contiguous run per (layer, K|V, head) and the attention kernel reads
    [block_size][dh] runs."""

    def __init__(self, spec: ModelSpec, n_blocks: int, block_size: int = 64, device="cuda") -> None:
        if block_size % 8:
            raise ValueError("block_size must be a multiple of 8")
        self.spec, self.block_size, self.n_blocks = spec, block_size, n_blocks
        self.slots = n_blocks * block_size
        numel = spec.layers * 2 * spec.kv_heads * self.slots * spec.head_dim
        # zero-initialised: the tensor-core attention reads whole 64-slot blocks and
        # masks positions past a sequence's length, so every slot must hold finite
        # values (0 * NaN would poison P.V); later contents are always written KV.
        self.data = torch.zeros(numel, dtype=torch.bfloat16, device=device)
        self._free: deque[int] = deque(range(n_blocks))
        # released blocks return to the free list only once the work enqueued before the
        # release has finished: several streams (serving, generation, peer copies) share
        # the pool, so stream order alone no longer protects a block's last readers
        self._pending: deque = deque()          # (event, blocks)
        self._lock = threading.Lock()
        self.reader_stream: torch.cuda.Stream | None = None  # where readers run (default: caller's stream)

    def blocks_for(self, n_tokens: int) -> int:
        return (n_tokens + self.block_size - 1) // self.block_size

    def alloc(self, n_tokens: int) -> list[int]:
        return self.alloc_blocks(self.blocks_for(n_tokens))

    def _reclaim(self, need: int) -> None:
        while self._pending and (len(self._free) < need or self._pending[0][0].query()):
            ev, blocks = self._pending.popleft()
            ev.synchronize()
            self._free.extend(blocks)

    def alloc_blocks(self, n: int) -> list[int]:
        with self._lock:
            self._reclaim(n)
            if n > len(self._free):
                raise MemoryError(f"KV pool exhausted: need {n} blocks, {len(self._free)} free")
            return [self._free.popleft() for _ in range(n)]

    def release(self, blocks: Sequence[int]) -> None:
        if not len(blocks):
            return
        if self.data.is_cuda:
            ev = torch.cuda.Event()
            ev.record(self.reader_stream or torch.cuda.current_stream(self.data.device))
            with self._lock:
                self._pending.append((ev, list(blocks)))
        else:
            with self._lock:
                self._free.extend(blocks)

    @property
    def free_blocks(self) -> int:
        with self._lock:
            return len(self._free) + sum(len(b) for _, b in self._pending)

    def gather(self, blocks: Sequence[int], n_tokens: int) -> torch.Tensor:
        """[L][2][Hkv][n_tokens][dh] copy of a sequence's KV (tests/debug)."""
        s = self.spec
        v = self.data.view(s.layers, 2, s.kv_heads, self.slots, s.head_dim)
        idx = torch.tensor([b * self.block_size + i for b in blocks for i in range(self.block_size)][:n_tokens],
                           device=self.data.device)
        return v.index_select(3, idx)


# ----------------------------------------------------------------- batch plans


@dataclass
class SeqPlan:
    tokens: np.ndarray          # new tokens (int32)
    n_cached: int               # cached-prefix tokens already in the pool
    blocks: Sequence[int]       # pool blocks covering positions [0, n_cached + len(tokens))


class BatchPlan:
    """Device metadata for rdkv_forward, packed into one int32 buffer (one H2D)."""

    def __init__(self, seqs: Sequence[SeqPlan], block_size: int, device) -> None:
        S = len(seqs)
        n_new = np.array([len(s.tokens) for s in seqs], dtype=np.int32)
        T = int(n_new.sum())
        if S == 0 or T == 0:
            raise ValueError("empty batch")
        bt_stride = max(len(s.blocks) for s in seqs)
        starts = np.zeros(S, np.int32)
        starts[1:] = np.cumsum(n_new)[:-1]
        cached = np.array([s.n_cached for s in seqs], dtype=np.int32)
        bt = np.zeros((S, bt_stride), np.int32)
        pos = np.empty(T, np.int32)
        slot = np.empty(T, np.int32)
        for i, s in enumerate(seqs):
            blk = np.asarray(s.blocks, dtype=np.int64)
            need = (s.n_cached + len(s.tokens) + block_size - 1) // block_size
            if len(blk) < need:
                raise ValueError(f"sequence {i}: {len(blk)} blocks cannot hold {s.n_cached + len(s.tokens)} tokens")
            bt[i, : len(blk)] = blk
            p = np.arange(s.n_cached, s.n_cached + len(s.tokens), dtype=np.int64)
            a, b = starts[i], starts[i] + len(s.tokens)
            pos[a:b] = p
            slot[a:b] = blk[p // block_size] * block_size + p % block_size
        last = starts + n_new - 1
        toks = np.concatenate([np.asarray(s.tokens, dtype=np.int32) for s in seqs])
        parts = [toks, pos, slot, starts, n_new, cached, bt.ravel(), last]
        offs = np.cumsum([0] + [len(p) for p in parts])
        host = torch.from_numpy(np.concatenate(parts).astype(np.int32))
        if torch.cuda.is_available():
            host = host.pin_memory()
        self.host = host
        self._offs = offs
        self.n_seqs, self.n_tokens, self.max_new = S, T, int(n_new.max())
        self.bt_stride, self.block_size = bt_stride, block_size
        self.n_new, self.n_cached = n_new, cached
        self.max_ctx = int((n_new + cached).max())
        self.flags = 0
        self.rebase(host.to(device, non_blocking=True))

    _FIELDS = ("tokens", "pos", "slot", "seq_start", "seq_new", "seq_cached", "block_table", "last_row")

    def rebase(self, meta: torch.Tensor) -> None:
        """Point the batch at a device copy of the metadata (a graph's static buffer)."""
        self.meta = meta
        base = meta.data_ptr()
        self.ptr = {k: base + 4 * int(o) for k, o in zip(self._FIELDS, self._offs[:-1])}

    def signature(self) -> tuple:
        # max_ctx fixes the split-KV choice baked into a captured graph
        return (self.n_seqs, self.n_tokens, self.max_new, self.bt_stride, self.block_size, self.max_ctx)

    def struct(self, kv_base: int, kv_slots: int, logits=None, next_token=None, layer_ready=None) -> RdkvBatch:
        p = self.ptr
        return RdkvBatch(
            n_seqs=self.n_seqs, n_tokens=self.n_tokens, max_new=self.max_new, block_size=self.block_size,
            bt_stride=self.bt_stride, want_logits=1 if logits is not None else 0,
            tokens=p["tokens"], pos=p["pos"], slot=p["slot"], seq_start=p["seq_start"], seq_new=p["seq_new"],
            seq_cached=p["seq_cached"], block_table=p["block_table"], last_row=p["last_row"],
            kv_base=kv_base, kv_slots=kv_slots,
            logits=logits.data_ptr() if logits is not None else None,
            next_token=next_token.data_ptr() if next_token is not None else None, max_ctx=self.max_ctx,
            layer_ready=C.cast(layer_ready, C.c_void_p).value if layer_ready is not None else None,
            flags=self.flags)


# ----------------------------------------------------------------- the model handle


class DeviceModel:
    """Owns an rdkv_model handle over device-resident weights."""

    def __init__(self, weights: ModelWeights, fold_norms: bool = True) -> None:
        s = weights.spec
        self.spec, self.weights = s, weights
        self.device = weights.embed.device
        if fold_norms:
            fold_norm_gains(weights)
        desc = RdkvModelDesc(layers=s.layers, hidden=s.hidden, n_heads=s.n_heads, kv_heads=s.kv_heads,
                             head_dim=s.head_dim, ffn=s.ffn, vocab=s.vocab, max_pos=s.max_pos,
                             rope_theta=s.rope_theta, norm_eps=s.norm_eps,
                             flags=RDKV_MODEL_NORM_FOLDED if fold_norms else 0)
        ptrs = weights.pointer_list()
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(_L().rdkv_model_create(C.byref(desc), arr, len(ptrs), C.byref(h)))
        self._h = h
        self._ws: dict | None = None

    def close(self) -> None:
        if self._h:
            _L().rdkv_model_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def workspace(self, n_tokens: int, n_seqs: int, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """Scratch for one forward; one buffer per stream, so forwards on different
        streams (serving and queue-time generation) never share scratch."""
        need = int(_L().rdkv_workspace_bytes(self._h, n_tokens, n_seqs))
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self._ws is None:
            self._ws = {}
        ws = self._ws.get(st.cuda_stream)
        if ws is None or ws.numel() < need:
            with torch.cuda.stream(st):
                ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            self._ws[st.cuda_stream] = ws
        return ws

    def profile(self, on: bool) -> None:
        _lib.check(_L().rdkv_profile_enable(self._h, 1 if on else 0))

    def collect(self) -> dict[str, dict]:
        """Per kernel class since the last collect: device ms, launches, GEMM FLOPs."""
        k = len(PROF_CLASSES)
        ms, n, fl = (C.c_double * k)(), (C.c_int64 * k)(), (C.c_double * k)()
        _lib.check(_L().rdkv_profile_collect(self._h, ms, n, fl))
        return {k: {"ms": ms[i], "launches": int(n[i]), "flops": fl[i]} for i, k in enumerate(PROF_CLASSES)}

    def forward(self, plan: BatchPlan, kv_base: int, kv_slots: int, logits=None, next_token=None,
                stream: torch.cuda.Stream | None = None, layer_ready=None) -> None:
        ws = self.workspace(plan.n_tokens, plan.n_seqs, stream)
        b = plan.struct(kv_base, kv_slots, logits, next_token, layer_ready)
        _lib.check(_L().rdkv_forward(self._h, C.byref(b), ws.data_ptr(), ws.numel(), _stream_ptr(stream)))


def fold_norm_gains(w: ModelWeights) -> None:
    """Fold the attention / MLP RMSNorm gains into the columns of w_qkv / w_gate_up
    (W'[n, k] = bf16(W[n, k] * gain[k])) in place and replace the gains by ones, so
    the weights describe the same function with unit-gain norms (the oracle reads
    them the same way).  The device then fuses each norm across its GEMMs
    (RDKV_MODEL_NORM_FOLDED).  Idempotent: folded gains are exactly 1."""
    for lw in w.layers:
        for wk, gk in (("wqkv", "attn_norm"), ("wgu", "mlp_norm")):
            g = lw[gk]
            if bool((g == 1).all()):
                continue
            W = lw[wk]
            for r0 in range(0, W.shape[0], 4096):  # bounded fp32 temporaries
                blk = W[r0:r0 + 4096]
                blk.copy_((blk.float() * g.float()[None, :]).to(W.dtype))
            lw[gk] = torch.ones_like(g)  # new tensor: gains shared with other shards stay intact


def kv_unpack(pool: KvPool, jobs: Sequence[tuple[torch.Tensor, int, int]], block_table: torch.Tensor,
              elem_width: int = 2, stream: torch.cuda.Stream | None = None, layers: tuple[int, int] | None = None,
              jobs_dev: torch.Tensor | None = None, heads: tuple[int, int] | None = None) -> None:
    """K3: unpack device-resident blob payloads into the pool.

    ``jobs`` = (payload device tensor, n_tokens, first_block index into the flat
    ``block_table`` int32 device tensor).  ``heads`` = (first head, heads in the
    payload) when the payloads hold more KV heads than the pool — a
    tensor-parallel rank reading its share of full-model blobs."""
    if not jobs:
        return
    if jobs_dev is None:
        jobs_dev = pack_unpack_jobs(jobs).to(pool.data.device, non_blocking=True)
    s = pool.spec
    l0, l1 = layers if layers is not None else (0, s.layers)
    h0, src_heads = heads if heads is not None else (0, s.kv_heads)
    _lib.check(_L().rdkv_kv_unpack_heads(jobs_dev.data_ptr(), len(jobs), max(n for _, n, _ in jobs),
                                         block_table.data_ptr(), pool.block_size, pool.data.data_ptr(), s.layers,
                                         s.kv_heads, s.head_dim, pool.slots, elem_width, l0, l1, h0, src_heads,
                                         _stream_ptr(stream)))
    # the job table may have been staged on another stream: keep its memory until this launch has read it
    jobs_dev.record_stream(stream if stream is not None else torch.cuda.current_stream(pool.data.device))


class LayerStreamer:
    """Layer-wise KV streaming.

    The payload layout puts the layer outermost, so layer l of every cached
    blob is one contiguous slice.  Per layer: (1) the host-tier slices are
    copied H2D on a copy stream, (2) K3 unpacks that layer on an unpack stream
    once its copy has landed and records event l, (3) the forward waits on
    event l only before layer l's attention.  PCIe transfer, the HBM-bound
    unpack and the compute-bound GEMMs of earlier layers all overlap."""

    def __init__(self, engine: "Engine") -> None:
        L = engine.spec.layers
        self.eng = engine
        self.stream = torch.cuda.Stream(device=engine.device)       # unpack
        self.h2d = torch.cuda.Stream(device=engine.device)          # host -> HBM copies
        self.events = [torch.cuda.Event() for _ in range(L)]
        self.copied = [torch.cuda.Event() for _ in range(L)]
        # layers per H2D copy: 2 measured best (C2: 94% of the pinned-copy peak vs 92% at 1,
        # 88% at 16 — fewer, larger DMAs, still early enough for the first attention)
        self.copy_layers = max(1, int(os.environ.get("RDKV_H2D_LAYERS", "2")))
        self.handles = (C.c_void_p * L)()
        self.copied_handles = (C.c_void_p * L)()
        # pinned host payloads whose raw cudaMemcpyAsync copies may still be reading
        # them: held until an event after the last copy has completed (the copies bypass
        # torch's CachingHostAllocator, which would otherwise recycle the block early)
        self._in_flight: deque = deque()
        # torch creates CUDA events lazily: record each once so the native call gets real handles
        cur = torch.cuda.current_stream(engine.device)
        for l in range(L):
            self.events[l].record(cur)
            self.copied[l].record(cur)
            self.handles[l] = self.events[l].cuda_event
            self.copied_handles[l] = self.copied[l].cuda_event

    def launch(self, pool: KvPool, jobs, block_table: torch.Tensor, jobs_dev: torch.Tensor, main: torch.cuda.Stream,
               first_event=None, last_event=None, h2d: Sequence[tuple[torch.Tensor, torch.Tensor]] = (),
               heads: tuple[int, int] | None = None):
        """Enqueue per-layer [H2D ->] unpack; returns the event-handle array for rdkv_forward.
        ``h2d`` = (pinned host payload, device staging buffer) pairs still to be copied."""
        L = len(self.events)
        self.stream.wait_stream(main)
        # buffers allocated on `main` but read here must not be recycled early
        jobs_dev.record_stream(self.stream)
        block_table.record_stream(self.stream)
        for src, _, _ in jobs:
            src.record_stream(self.stream)
        if h2d:
            self.h2d.wait_stream(main)
            for _, dev in h2d:
                dev.record_stream(self.h2d)
        if first_event is not None:
            first_event.record(self.stream)
        if not jobs:  # nothing to move: the layer events complete at once
            for ev in self.events:
                ev.record(self.stream)
            if last_event is not None:
                last_event.record(self.stream)
            return self.handles
        # the whole per-layer [H2D ->] unpack -> event chain is enqueued by one native call
        # (enqueueing it from Python cost ~0.7 ms of host time per query, which delayed the
        # forward's launch behind the copies it overlaps with)
        s = pool.spec
        h0, src_heads = heads if heads is not None else (0, s.kv_heads)
        n = len(h2d)
        hosts = (C.c_void_p * max(n, 1))(*[host.data_ptr() for host, _ in h2d])
        devs = (C.c_void_p * max(n, 1))(*[dev.data_ptr() for _, dev in h2d])
        per = (C.c_size_t * max(n, 1))(*[host.numel() * host.element_size() // L for host, _ in h2d])
        _lib.check(_L().rdkv_kv_stream_layers(
            jobs_dev.data_ptr(), len(jobs), max(nt for _, nt, _ in jobs), block_table.data_ptr(), pool.block_size,
            pool.data.data_ptr(), s.layers, s.kv_heads, s.head_dim, pool.slots, 2, h0, src_heads, n, hosts, devs,
            per, self.copy_layers, _stream_ptr(self.h2d), _stream_ptr(self.stream), self.copied_handles,
            self.handles))
        if h2d:
            self._hold([host for host, _ in h2d])
        if last_event is not None:
            last_event.record(self.stream)
        return self.handles


    def _hold(self, hosts) -> None:
        while self._in_flight and self._in_flight[0][0].query():
            self._in_flight.popleft()
        done = torch.cuda.Event()
        done.record(self.h2d)
        self._in_flight.append((done, hosts))


def pack_unpack_jobs(jobs: Sequence[tuple[torch.Tensor, int, int]]) -> torch.Tensor:
    arr = np.zeros(len(jobs), dtype=_UNPACK_DTYPE)
    for i, (src, n, fb) in enumerate(jobs):
        arr[i] = (src.data_ptr(), n, fb, 0)
    host = torch.from_numpy(arr.view(np.uint8).copy())
    return host.pin_memory() if torch.cuda.is_available() else host


class _Graph:
    __slots__ = ("graph", "meta", "jobs", "logits", "nxt", "ws", "plan")


class GraphRunner:
    """CUDA-graph replay of [K3 unpack ->] rdkv_forward for a fixed batch shape.

    A serving step is ~7 launches per layer; for small batches (single-query
    TTFT) host launch overhead dominates.  Each distinct shape (sequences,
    tokens, block-table width, unpack jobs) is captured once with static
    metadata / job / output buffers; replays only copy the new metadata in."""

    MAX_TOKENS = 16384

    def __init__(self, engine: "Engine", max_entries: int = 8) -> None:
        self.eng = engine
        self.max_entries = max_entries
        self._cache: "OrderedDict[tuple, _Graph]" = OrderedDict()

    def run(self, plan: BatchPlan, jobs, want_logits: bool = True):
        if plan.n_tokens > self.MAX_TOKENS:
            return None
        key = plan.signature() + (len(jobs), max((n for _, n, _ in jobs), default=0), want_logits)
        e = self._cache.get(key)
        jobs_host = pack_unpack_jobs(jobs) if jobs else None
        if e is None:
            e = self._build(plan, jobs, jobs_host, key, want_logits)
        else:
            self._cache.move_to_end(key)
            e.meta.copy_(plan.host, non_blocking=True)
            if jobs_host is not None:
                e.jobs.copy_(jobs_host, non_blocking=True)
            e.graph.replay()
        return e.logits, e.nxt

    def _build(self, plan, jobs, jobs_host, key, want_logits) -> _Graph:
        eng, s = self.eng, self.eng.spec
        dev = eng.device
        e = _Graph()
        e.meta = torch.empty(plan.host.numel(), dtype=torch.int32, device=dev)
        e.meta.copy_(plan.host, non_blocking=True)
        plan.rebase(e.meta)
        e.plan = plan
        e.jobs = None
        if jobs_host is not None:
            e.jobs = torch.empty(jobs_host.numel(), dtype=torch.uint8, device=dev)
            e.jobs.copy_(jobs_host, non_blocking=True)
        e.logits = torch.empty(plan.n_seqs, s.vocab, dtype=torch.float32, device=dev) if want_logits else None
        e.nxt = torch.empty(plan.n_seqs, dtype=torch.int32, device=dev) if want_logits else None
        nbytes = int(_L().rdkv_workspace_bytes(eng.model._h, plan.n_tokens, plan.n_seqs))
        e.ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        pool = eng.pool
        n_jobs = len(jobs)
        max_tok = max((n for _, n, _ in jobs), default=0)
        bt_ptr = plan.ptr["block_table"]

        bt_view = plan.meta[(bt_ptr - plan.meta.data_ptr()) // 4:]

        def body():
            main = torch.cuda.current_stream()
            handles = None
            if n_jobs:
                handles = eng.streamer.launch(pool, jobs, bt_view, e.jobs, main)
            b = plan.struct(pool.data.data_ptr(), pool.slots, e.logits, e.nxt, handles)
            _lib.check(_L().rdkv_forward(eng.model._h, C.byref(b), e.ws.data_ptr(), e.ws.numel(), main.cuda_stream))

        body()  # eager warm-up (first launches set kernel attributes) and this call's result
        torch.cuda.current_stream().synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        e.graph = g
        self._cache[key] = e
        if len(self._cache) > self.max_entries:
            self._cache.popitem(last=False)
        return e


# ----------------------------------------------------------------- the instance


@dataclass
class QueryRequest:
    """One query: a cached prefix (device payload, or None) plus new tokens."""

    new_tokens: np.ndarray
    cached_payload: torch.Tensor | None = None   # device bf16 payload [L][2][Hkv][n_cached][dh]
    n_cached: int = 0


@dataclass
class ResidentEntry:
    blocks: list[int]       # pool blocks holding positions [0, n_tokens)
    n_tokens: int
    pins: int = 0           # batches currently reading the blocks
    ready: object = None    # CUDA event after which the blocks hold the KV (None: already complete)


class ResidentKvTier:
    """HBM tier: KvKey -> cached prefix KV living *in the paged pool* (block-LRU).

    A hit costs nothing to load: the query's block table starts with the
    entry's blocks and only its new tokens get fresh blocks (a partial last
    block is copied on write).  Entries are filled once, by one K3 unpack of
    the blob payload, when a composite is generated or first streamed in.

    Prefixes share blocks: the KV of prefix ``doc_ids[:j]`` is exactly the
    first rows of its combination's KV (causal attention, row-deterministic
    kernels — SURVEY H-e), so :meth:`alias` makes all k prefix keys of a
    resident combination resident at the cost of the combination alone.
    Blocks are reference-counted; an entry's eviction frees only blocks no
    other entry shares.

    Purely a *placement* layer: what the store holds and how it accounts an
    access is unchanged; this only changes where the bytes come from (SURVEY
    §8e invariant).  ``can_evict(key)`` (the control plane's retract) vetoes
    evicting an entry a peer is still copying over NVLink."""

    def __init__(self, pool: "KvPool", capacity_blocks: int) -> None:
        self.pool = pool
        self.capacity = capacity_blocks
        self._d: "OrderedDict[object, ResidentEntry]" = OrderedDict()
        self._ref: dict[int, int] = {}
        self._reserved = 0
        self._lock = threading.Lock()
        self.can_evict = None
        self.evictions = 0

    @property
    def used(self) -> int:
        return len(self._ref) + self._reserved

    def __contains__(self, key) -> bool:
        with self._lock:
            return key in self._d

    def __len__(self) -> int:
        return len(self._d)

    def items(self) -> list:
        with self._lock:
            return list(self._d.items())

    def get(self, key) -> ResidentEntry | None:
        with self._lock:
            return self._d.get(key)

    def acquire(self, key) -> ResidentEntry | None:
        """Pin and return the entry (MRU), or None."""
        with self._lock:
            e = self._d.get(key)
            if e is not None:
                self._d.move_to_end(key)
                e.pins += 1
            return e

    def unpin(self, key) -> None:
        with self._lock:
            e = self._d.get(key)
            if e is not None and e.pins > 0:
                e.pins -= 1

    def _drop(self, key) -> list[int]:
        e = self._d.pop(key)
        freed = []
        for b in e.blocks:
            r = self._ref[b] - 1
            if r:
                self._ref[b] = r
            else:
                del self._ref[b]
                freed.append(b)
        self.evictions += 1
        return freed

    def reserve(self, n_tokens: int) -> list[int] | None:
        """Blocks for a new entry, evicting unpinned LRU entries; None if it cannot fit."""
        need = self.pool.blocks_for(n_tokens)
        freed: list[int] = []
        with self._lock:
            if need > self.capacity:
                return None
            for k in list(self._d):
                if self.used + need <= self.capacity:
                    break
                e = self._d[k]
                if e.pins or (self.can_evict is not None and not self.can_evict(k)):
                    continue
                freed += self._drop(k)
            ok = self.used + need <= self.capacity
            if ok:
                self._reserved += need
        self.pool.release(freed)
        if not ok:
            return None
        try:
            return self.pool.alloc_blocks(need)
        except MemoryError:
            with self._lock:
                self._reserved -= need
            return None

    def unreserve(self, blocks: list[int]) -> None:
        with self._lock:
            self._reserved -= len(blocks)
        self.pool.release(blocks)

    def commit(self, key, blocks: list[int], n_tokens: int, ready=None) -> bool:
        """Publish reserved ``blocks`` as ``key``'s entry.  If another writer got there
        first, the existing entry wins (a batch may have it pinned and be reading
        its blocks) and the new blocks go back to the pool.  False in that case."""
        with self._lock:
            self._reserved -= len(blocks)
            if key in self._d:
                lost = True
            else:
                lost = False
                for b in blocks:
                    self._ref[b] = self._ref.get(b, 0) + 1
                self._d[key] = ResidentEntry(list(blocks), n_tokens, ready=ready)
        if lost:
            self.pool.release(blocks)
        return not lost

    def alias(self, key, base_key, n_tokens: int) -> bool:
        """Make ``key`` resident as the first ``n_tokens`` positions of ``base_key``'s
        entry (its leading blocks, shared).  False if the base is not resident."""
        with self._lock:
            if key in self._d:
                return True
            base = self._d.get(base_key)
            if base is None or n_tokens > base.n_tokens:
                return False
            blocks = base.blocks[: self.pool.blocks_for(n_tokens)]
            for b in blocks:
                self._ref[b] += 1
            self._d[key] = ResidentEntry(list(blocks), n_tokens, ready=base.ready)
            return True

    def clear(self) -> int:
        """Evict every unpinned entry; returns how many were dropped."""
        keys = [k for k, _ in self.items()]
        return sum(self.evict(k) for k in keys)

    def evict(self, key) -> bool:
        """Drop ``key`` (if unpinned); its unshared blocks return to the pool."""
        with self._lock:
            e = self._d.get(key)
            if e is None or e.pins:
                return False
            freed = self._drop(key)
        self.pool.release(freed)
        return True


class Engine:
    """Model instance bound to one GPU."""

    def __init__(self, spec: ModelSpec, weights: ModelWeights | None = None, seed: int = 0, device="cuda",
                 pool_tokens: int = 1 << 16, block_size: int = 64, device_cache_bytes: int = 0) -> None:
        """``pool_tokens`` = working KV slots for in-flight queries; ``device_cache_bytes``
        = extra pool capacity reserved for the HBM-resident tier of cached prefixes."""
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.spec = spec
        self.weights = weights if weights is not None else init_weights(spec, seed, self.device)
        self.model = DeviceModel(self.weights)
        work_blocks = (pool_tokens + block_size - 1) // block_size
        block_bytes = spec.kv_bytes_per_token() * block_size
        tier_blocks = device_cache_bytes // block_bytes
        self.pool = KvPool(spec, work_blocks + tier_blocks, block_size, self.device)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.resident = ResidentKvTier(self.pool, tier_blocks)
        self.tp_rank = 0  # set by multi.TpGroup: which KV heads of full-model blobs this rank owns
        self.graphs = GraphRunner(self)
        self.streamer = LayerStreamer(self)

    def stage(self, payload: torch.Tensor, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """Async H2D copy of a pinned host payload; returns the device bf16 view."""
        dev = torch.empty(payload.numel(), dtype=torch.uint8, device=self.device)
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            dev.copy_(payload, non_blocking=True)
        return dev.view(torch.bfloat16)

    def make_resident(self, key, payload: torch.Tensor, n_tokens: int,
                      stream: torch.cuda.Stream | None = None) -> bool:
        """Place a device blob payload [L][2][Hkv][n][dh] into the HBM tier (one K3
        unpack into freshly reserved pool blocks).  False if it does not fit."""
        if key in self.resident:
            return True
        blocks = self.resident.reserve(n_tokens)
        if blocks is None:
            return False
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            bt = torch.tensor(blocks, dtype=torch.int32).pin_memory().to(self.device, non_blocking=True)
        kv_unpack(self.pool, [(payload, n_tokens, 0)], bt, stream=s)
        payload.record_stream(s)
        bt.record_stream(s)
        ready = torch.cuda.Event()
        ready.record(s)
        self.resident.commit(key, blocks, n_tokens, ready=ready)
        return True

    def copy_block(self, src_block: int, dst_block: int, n_tokens: int,
                   stream: torch.cuda.Stream | None = None) -> None:
        s = self.spec
        _lib.check(_L().rdkv_kv_copy_block(self.pool.data.data_ptr(), s.layers, s.kv_heads, s.head_dim,
                                           self.pool.slots, self.pool.block_size, src_block, dst_block, n_tokens,
                                           _stream_ptr(stream)))

    # -------------------------------------------------------------- generation
    def generate_doc_kv(self, tokens: np.ndarray, out: torch.Tensor | None = None,
                        stream: torch.cuda.Stream | None = None, row_deterministic: bool = True) -> torch.Tensor:
        """Document KV of ``tokens`` (positions 0..n-1) in the blob payload layout
        [L][2][Hkv][n][dh] bf16, as a flat device tensor.  ``row_deterministic``
        keeps every row's arithmetic independent of n (no split-KV attention for
        short documents), so the KV of a prefix is bit-identical to the same rows
        of a longer combination's KV (SURVEY H-e)."""
        s, n = self.spec, len(tokens)
        numel = s.layers * 2 * s.kv_heads * n * s.head_dim
        if out is None:
            out = torch.empty(numel, dtype=torch.bfloat16, device=self.device)
        plan = BatchPlan([SeqPlan(np.asarray(tokens, np.int32), 0, [0])], block_size=n, device=self.device)
        if row_deterministic:
            plan.flags |= 1  # RDKV_BATCH_ROW_DETERMINISTIC
        self.model.forward(plan, out.data_ptr(), n, stream=stream)
        plan.meta.record_stream(stream if stream is not None else torch.cuda.current_stream(self.device))
        return out

    # -------------------------------------------------------------- query prefill
    def prefill(self, requests: Sequence[QueryRequest], stream: torch.cuda.Stream | None = None):
        """Batched prefill over cached prefixes -> (logits [S,V] fp32, next_token [S] int32)."""
        pool = self.pool
        seqs, owned = [], []
        try:
            for r in requests:
                blocks = pool.alloc(r.n_cached + len(r.new_tokens))
                owned.append(blocks)
                seqs.append(SeqPlan(np.asarray(r.new_tokens, np.int32), r.n_cached, blocks))
            plan = BatchPlan(seqs, pool.block_size, self.device)
            jobs = [(r.cached_payload, r.n_cached, i * plan.bt_stride)
                    for i, r in enumerate(requests) if r.n_cached > 0]
            if jobs:
                kv_unpack(pool, jobs, _bt_view(plan), stream=stream)
            S = len(requests)
            logits = torch.empty(S, self.spec.vocab, dtype=torch.float32, device=self.device)
            nxt = torch.empty(S, dtype=torch.int32, device=self.device)
            self.model.forward(plan, pool.data.data_ptr(), pool.slots, logits, nxt, stream=stream)
            return logits, nxt
        finally:
            for b in owned:
                pool.release(b)


def _bt_view(plan: BatchPlan) -> torch.Tensor:
    off = (plan.ptr["block_table"] - plan.meta.data_ptr()) // 4
    return plan.meta[off: off + plan.n_seqs * plan.bt_stride]
