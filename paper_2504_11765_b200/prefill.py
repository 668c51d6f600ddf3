"""Prefill-with-cached-prefix: the measured counterpart of ``costs.ttft``.

Reference semantics (costs.py:121-144, sim.py:414-436): the longest cached
prefix of the query's ordered document combination is loaded from the tier
the lookup reports, and only the *new* tokens — the uncached documents, then
the query (sim.py:420-422) — are prefilled, attending over the whole context
(costs.py:89-99).  On a MISS the would-be-cached tokens are plain text and join
the prefill (costs.py:136-138).

Here the load is real (pinned host payload -> HBM on a side stream, then the
K3 unpack into the paged pool; or nothing at all when the prefix is already
resident in the pool's HBM tier) and
so is the prefill (tcgen05 GEMMs + attention + LM head).  Both halves are
timed with CUDA events and returned as the reference's
``(seconds, TtftBreakdown(kv_load, prefill))`` plus the first-token logits.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from .costs import TtftBreakdown
from .engine import BatchPlan, Engine, SeqPlan, _bt_view, kv_unpack, pack_unpack_jobs
from .store import KvKey, LookupResult, Outcome


@dataclass
class PrefillRequest:
    lookup: LookupResult              # outcome of store.get for the longest cached prefix (MISS if none)
    prefix_tokens: np.ndarray         # tokens of that prefix combination (raw text on a miss)
    new_tokens: np.ndarray            # remaining documents, then the query
    key: KvKey | None = None          # enables the HBM placement cache


@dataclass
class LiveSequence:
    """A prefilled sequence kept alive for decoding (``prefill_batch(keep=True)``): its pool
    blocks hold the KV of positions [0, n_ctx); ``owned`` are the blocks it allocated
    (released by ``decode.retire``), ``pinned`` the HBM-tier entry whose blocks it shares."""
    blocks: list
    owned: list
    n_ctx: int
    pinned: KvKey | None = None


@dataclass
class PrefillResult:
    ttft: float
    breakdown: TtftBreakdown
    logits: torch.Tensor              # [S, V] fp32 on the device
    next_token: torch.Tensor          # [S] int32 on the device
    sequences: list | None = None     # LiveSequence per request when keep=True


def prefill_batch(engine: Engine, requests: Sequence[PrefillRequest], timed: bool = True,
                  unpack_events: list | None = None, use_graph: bool = True,
                  stream_layers: bool = True, keep: bool = False) -> PrefillResult:
    """Serve a batch of queries on one engine; kv_load / prefill are the
    device-measured durations of the whole batch's load and prefill phases.
    ``unpack_events`` collects (start, end) CUDA events around the K3 launch.
    Untimed calls replay a per-shape CUDA graph (``Engine.graphs``); its output
    tensors are reused by the next call of the same shape.  ``keep`` hands every
    sequence's pool blocks (and its HBM-tier pin) to the caller as
    ``result.sequences`` for decoding (``decode.py``) instead of releasing them."""
    pool = engine.pool
    main = torch.cuda.current_stream(engine.device)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if timed else None
    if timed:
        ev[0].record(main)
    seqs, owned, jobs, staged, pending_h2d, pinned = [], [], [], [], [], []
    pin_of: dict[int, KvKey] = {}
    kept = False
    bs = pool.block_size
    # staging buffers are allocated on `main`; the copy stream must not write
    # them before main's earlier users of that memory are done
    engine.copy_stream.wait_stream(main)
    try:
        for i, r in enumerate(requests):
            hit = r.lookup.outcome is not Outcome.MISS
            new = np.asarray(r.new_tokens, np.int32) if hit else np.concatenate(
                [np.asarray(r.prefix_tokens, np.int32), np.asarray(r.new_tokens, np.int32)])
            entry = engine.resident.acquire(r.key) if hit and r.key is not None else None
            if entry is not None:
                pinned.append(r.key)
                pin_of[i] = r.key
            if hit and r.lookup.blob is None and entry is None:
                raise ValueError(f"request {i}: an HBM-tier hit needs the prefix resident in the pool")
            n_cached = (entry.n_tokens if r.lookup.blob is None else int(r.lookup.blob.header.token_count)) \
                if hit else 0
            if entry is not None:
                # HBM-tier hit: the prefix is already in pool blocks; only the new
                # tokens get fresh blocks (a partial last block is copied on write)
                if entry.ready is not None:  # filled on another stream (queue-time generation, peer fetch)
                    main.wait_event(entry.ready)
                if entry.n_tokens != n_cached:
                    raise ValueError("resident entry does not match the lookup's token count")
                prefix = list(entry.blocks)
                tail = n_cached % bs
                fresh = pool.alloc_blocks(pool.blocks_for(n_cached + len(new)) - len(prefix) + (1 if tail else 0))
                owned.append(fresh)
                if tail:
                    engine.copy_block(prefix[-1], fresh[0], tail, stream=main)
                    prefix[-1] = fresh[0]
                    fresh = fresh[1:]
                seqs.append(SeqPlan(new, n_cached, prefix + fresh))
                continue
            blocks = pool.alloc(n_cached + len(new))
            owned.append(blocks)
            seqs.append(SeqPlan(new, n_cached, blocks))
            if hit:
                host = r.lookup.blob.payload_tensor()
                dev_copy = r.lookup.blob.device
                if dev_copy is not None and dev_copy.device == engine.device:  # already in HBM (GPU-verified disk hit)
                    dev = dev_copy.view(torch.bfloat16)
                    staged.append(dev)
                    jobs.append((dev, n_cached, i))
                    continue
                if stream_layers and not timed:  # copied layer by layer by the streamer
                    dev = torch.empty(host.numel(), dtype=torch.uint8, device=engine.device).view(torch.bfloat16)
                    pending_h2d.append((host, dev.view(torch.uint8)))
                else:
                    dev = engine.stage(host, stream=engine.copy_stream)
                staged.append(dev)
                jobs.append((dev, n_cached, i))
        # full-model blobs on a tensor-parallel rank: unpack only this rank's KV heads
        heads = None
        src = {int(requests[i].lookup.blob.header.kv_heads) for _, _, i in jobs}
        if len(src) > 1:
            raise ValueError("one batch mixes payloads with different KV-head counts")
        if src and src != {engine.spec.kv_heads}:
            (n_src,) = src
            heads = (engine.tp_rank * engine.spec.kv_heads, n_src)
        plan = BatchPlan(seqs, pool.block_size, engine.device)
        if staged:
            main.wait_stream(engine.copy_stream)
        ujobs = [(d, n, i * plan.bt_stride) for d, n, i in jobs]
        graphed = None
        if use_graph and not timed and unpack_events is None and not pending_h2d and heads is None:
            graphed = engine.graphs.run(plan, ujobs)  # [K3 unpack ->] forward as one CUDA-graph replay
        if graphed is not None:
            logits, nxt = graphed
            kv_load = prefill = 0.0
        else:
            handles = None
            if ujobs and stream_layers and not timed:
                # layer-wise streaming: per-layer unpacks on a side stream overlap the forward
                ua = ub = None
                if unpack_events is not None:
                    ua, ub = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    unpack_events.append((ua, ub))
                jobs_dev = pack_unpack_jobs(ujobs).to(engine.device, non_blocking=True)
                handles = engine.streamer.launch(pool, ujobs, _bt_view(plan), jobs_dev, main, ua, ub, h2d=pending_h2d,
                                                 heads=heads)
            elif ujobs:
                if unpack_events is not None:
                    ua, ub = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    ua.record(main)
                kv_unpack(pool, ujobs, _bt_view(plan), elem_width=2, stream=main, heads=heads)
                if unpack_events is not None:
                    ub.record(main)
                    unpack_events.append((ua, ub))
            if timed:
                ev[1].record(main)
            S = len(requests)
            logits = torch.empty(S, engine.spec.vocab, dtype=torch.float32, device=engine.device)
            nxt = torch.empty(S, dtype=torch.int32, device=engine.device)
            engine.model.forward(plan, pool.data.data_ptr(), pool.slots, logits, nxt, stream=main,
                                 layer_ready=handles)
            if timed:
                ev[2].record(main)
                ev[2].synchronize()
                kv_load = ev[0].elapsed_time(ev[1]) / 1e3
                prefill = ev[1].elapsed_time(ev[2]) / 1e3
            else:
                kv_load = prefill = 0.0
        for d in staged:  # keep staging buffers alive until the stream has consumed them
            d.record_stream(main)
        bd = TtftBreakdown(kv_load, prefill)
        live = None
        if keep:
            live = [LiveSequence(list(sp.blocks), list(own), int(sp.n_cached + len(sp.tokens)), pin_of.get(i))
                    for i, (sp, own) in enumerate(zip(seqs, owned))]
            kept = True
        return PrefillResult(bd.total, bd, logits, nxt, live)
    finally:
        if not kept:
            for b in owned:
                pool.release(b)
            for k in pinned:
                engine.resident.unpin(k)


def prefill_with_cached_prefix(engine: Engine, lookup: LookupResult, prefix_tokens, new_tokens,
                               key: KvKey | None = None) -> tuple[float, TtftBreakdown, torch.Tensor, int]:
    """Single query: (ttft seconds, TtftBreakdown, logits [V], first token)."""
    r = prefill_batch(engine, [PrefillRequest(lookup, prefix_tokens, new_tokens, key)])
    return r.ttft, r.breakdown, r.logits[0], int(r.next_token[0])
