"""Decode phase after the first token, with continuous batching.

The reference has decoding only as a constant: ``CostParams.decode_enabled`` /
``decode_time_per_token`` (costs.py:62-71) adds ``decode_tokens x
decode_time_per_token`` to a batch's span in ``run_single_instance``
(sim.py:572-573).  Here the tokens are really generated on the B200: every
sequence keeps the pool blocks its prefill wrote (``prefill_batch(keep=True)``:
the cached prefix — shared, pinned HBM-tier blocks or the unpacked host/disk
payload — plus the new tokens), and each decode step is one ``rdkv_forward`` of
ONE new token per live sequence over its whole context (the same tcgen05 GEMMs,
paged attention and LM head + argmax as the prefill; the new token's K/V goes
straight into the sequence's next pool slot).  Greedy (argmax) decoding.

``ContinuousBatcher`` admits waiting requests between steps (their prefill is
one batched ``prefill_batch``), runs one step for every live sequence, and
retires sequences that produced their ``max_new_tokens`` — so requests join and
leave the running batch at token granularity.  ``decode_time_per_token``
measures the per-token step time of a batch for the reference's cost model.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from .engine import BatchPlan, Engine, SeqPlan
from .prefill import LiveSequence, PrefillRequest, prefill_batch


@dataclass
class DecodeSeq:
    """One sequence being decoded."""
    live: LiveSequence
    last: int                         # last generated token = the next step's input
    max_new: int                      # tokens to generate in total, the first one included
    tokens: list = field(default_factory=list)   # generated so far (the first token included)
    rid: int = -1                     # caller's id

    @property
    def done(self) -> bool:
        return len(self.tokens) >= self.max_new


def start(engine: Engine, requests: Sequence[PrefillRequest], max_new_tokens: int | Sequence[int],
          use_graph: bool = False) -> list[DecodeSeq]:
    """Prefill ``requests`` (cached-prefix semantics of prefill_batch) and keep their KV:
    one DecodeSeq per request holding its first token."""
    if not requests:
        return []
    mx = [max_new_tokens] * len(requests) if isinstance(max_new_tokens, int) else list(max_new_tokens)
    if any(m < 1 for m in mx):
        raise ValueError("max_new_tokens must be >= 1")
    r = prefill_batch(engine, requests, timed=False, use_graph=use_graph, keep=True)
    first = r.next_token.cpu().tolist()
    return [DecodeSeq(live, int(t), m, [int(t)]) for live, t, m in zip(r.sequences, first, mx)]


class _Step:
    """Reused device buffers for one decode step's logits / next tokens."""

    def __init__(self, engine: Engine) -> None:
        self.engine = engine
        self.cap = 0
        self.logits = self.nxt = None

    def buffers(self, n: int):
        if n > self.cap:
            self.cap = max(n, 2 * self.cap)
            e = self.engine
            self.logits = torch.empty(self.cap, e.spec.vocab, dtype=torch.float32, device=e.device)
            self.nxt = torch.empty(self.cap, dtype=torch.int32, device=e.device)
        return self.logits[:n], self.nxt[:n]


def _steps(engine: Engine) -> _Step:
    st = getattr(engine, "_decode_step", None)
    if st is None:
        st = engine._decode_step = _Step(engine)
    return st


def step(engine: Engine, seqs: Sequence[DecodeSeq], sync: bool = True,
         dev_tokens: torch.Tensor | None = None) -> torch.Tensor:
    """One decode step on the current stream: every sequence in ``seqs`` (not done) feeds
    its last token at position n_ctx and gets its next token.  Returns the [S] int32 next
    tokens on the device (a reused buffer).  With ``sync`` (default) they are copied to
    the host and appended to the sequences; without it, pass the previous step's result
    as ``dev_tokens`` (same sequences, same order) so the input tokens never leave the GPU."""
    act = [s for s in seqs if not s.done]
    if not act:
        return torch.empty(0, dtype=torch.int32)
    pool = engine.pool
    bs = pool.block_size
    plans = []
    for s in act:
        lv = s.live
        if lv.n_ctx + 1 > len(lv.blocks) * bs:  # the next slot opens a new block
            nb = pool.alloc_blocks(1)
            lv.blocks.extend(nb)
            lv.owned.extend(nb)
        plans.append(SeqPlan(np.array([s.last], np.int32), lv.n_ctx, lv.blocks))
    plan = BatchPlan(plans, bs, engine.device)
    if dev_tokens is not None:  # the tokens field leads the metadata buffer (BatchPlan._FIELDS)
        if dev_tokens.numel() != len(act):
            raise ValueError("dev_tokens must hold one token per live sequence")
        plan.meta[: len(act)].copy_(dev_tokens)
    logits, nxt = _steps(engine).buffers(len(act))
    nxt = nxt.clone() if dev_tokens is not None and dev_tokens.data_ptr() == nxt.data_ptr() else nxt
    engine.model.forward(plan, pool.data.data_ptr(), pool.slots, logits, nxt)
    for s in act:
        s.live.n_ctx += 1
    if sync:
        for s, t in zip(act, nxt.cpu().tolist()):
            s.last = int(t)
            s.tokens.append(int(t))
    else:
        for s in act:
            s.tokens.append(-1)  # placeholder: the token stays on the device
    return nxt


def extend(engine: Engine, parts: Sequence[tuple[LiveSequence, np.ndarray]]) -> torch.Tensor:
    """One forward that appends ``tokens`` to each live sequence — a decode step's single
    token, or the next chunk of a prompt being prefilled in chunks (chunked prefill: long
    prompts share forwards with the running decodes) — over the sequences' paged contexts.
    Returns the [S] int32 argmax after each sequence's last appended token (device)."""
    pool = engine.pool
    bs = pool.block_size
    plans = []
    for lv, toks in parts:
        need = (lv.n_ctx + len(toks) + bs - 1) // bs
        if need > len(lv.blocks):
            nb = pool.alloc_blocks(need - len(lv.blocks))
            lv.blocks.extend(nb)
            lv.owned.extend(nb)
        plans.append(SeqPlan(np.asarray(toks, np.int32), lv.n_ctx, lv.blocks))
    plan = BatchPlan(plans, bs, engine.device)
    logits, nxt = _steps(engine).buffers(len(parts))
    engine.model.forward(plan, pool.data.data_ptr(), pool.slots, logits, nxt)
    for lv, toks in parts:
        lv.n_ctx += len(toks)
    return nxt


def retire(engine: Engine, seq: DecodeSeq) -> None:
    """Release a finished (or abandoned) sequence's blocks and its HBM-tier pin."""
    lv = seq.live
    if lv.owned:
        engine.pool.release(lv.owned)
        lv.owned = []
    if lv.pinned is not None:
        engine.resident.unpin(lv.pinned)
        lv.pinned = None
    lv.blocks = []


def generate(engine: Engine, requests: Sequence[PrefillRequest], max_new_tokens: int) -> list[list[int]]:
    """Greedy generation of ``max_new_tokens`` per request (the first token included),
    all requests decoded as one batch."""
    seqs = start(engine, requests, max_new_tokens)
    try:
        while any(not s.done for s in seqs):
            step(engine, seqs)
        return [s.tokens for s in seqs]
    finally:
        for s in seqs:
            retire(engine, s)


class ContinuousBatcher:
    """Token-granular batching: ``submit`` queues requests; every ``tick`` admits up to
    ``max_batch - live`` waiting requests with one batched prefill (their first tokens),
    then runs one decode step for the sequences that were already live, and retires
    the finished ones (``finished`` maps request id -> generated tokens)."""

    def __init__(self, engine: Engine, max_batch: int = 32) -> None:
        self.engine = engine
        self.max_batch = max_batch
        self.waiting: list[tuple[int, PrefillRequest, int]] = []
        self.live: list[DecodeSeq] = []
        self.finished: dict[int, list[int]] = {}
        self.steps = 0
        self.prefills = 0
        self._next_id = 0

    def submit(self, request: PrefillRequest, max_new_tokens: int) -> int:
        rid = self._next_id
        self._next_id += 1
        self.waiting.append((rid, request, max_new_tokens))
        return rid

    def tick(self) -> None:
        room = self.max_batch - len(self.live)
        running = [s for s in self.live if not s.done]
        if self.waiting and room > 0:
            batch, self.waiting = self.waiting[:room], self.waiting[room:]
            new = start(self.engine, [r for _, r, _ in batch], [m for _, _, m in batch])
            for (rid, _, _), s in zip(batch, new):
                s.rid = rid
            self.live.extend(new)
            self.prefills += 1
        if running:
            step(self.engine, running)
            self.steps += 1
        keep = []
        for s in self.live:
            if s.done:
                self.finished[s.rid] = s.tokens
                retire(self.engine, s)
            else:
                keep.append(s)
        self.live = keep

    def run(self) -> dict[int, list[int]]:
        """Tick until every submitted request has finished."""
        while self.waiting or self.live:
            self.tick()
        return self.finished

    def close(self) -> None:
        for s in self.live:
            retire(self.engine, s)
        self.live = []


def decode_time_per_token(engine: Engine, requests: Sequence[PrefillRequest], n_steps: int = 16) -> dict:
    """Measure the decode step of a batch (CUDA events around ``n_steps`` steps after the
    prefill): seconds per step, per generated token, and tokens/s — the calibration of the
    reference's ``CostParams.decode_time_per_token`` (costs.py:70-71)."""
    seqs = start(engine, requests, n_steps + 2)
    try:
        step(engine, seqs)  # warm-up step
        main = torch.cuda.current_stream(engine.device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        prev = torch.tensor([s.last for s in seqs], dtype=torch.int32, device=engine.device)
        e0.record(main)
        for _ in range(n_steps):
            prev = step(engine, seqs, sync=False, dev_tokens=prev).clone()
        e1.record(main)
        e1.synchronize()
        dt = e0.elapsed_time(e1) / 1e3 / n_steps
        return {"seconds_per_step": dt, "batch": len(seqs), "seconds_per_token": dt / len(seqs),
                "tokens_per_s": len(seqs) / dt, "steps": n_steps}
    finally:
        for s in seqs:
            retire(engine, s)
