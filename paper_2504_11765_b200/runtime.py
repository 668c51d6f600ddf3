"""Real-time multi-instance serving with queue-time proactive KV precompute.

The reference models this system as a discrete-event simulation (``sim.run``,
sim.py:358-504): one central FIFO dispatched to idle instances
(sim.py:403-409), the longest cached prefix of each query's ordered document
combination loaded and the rest prefilled (sim.py:414-436), and a generator
that precomputes the missing prefixes of any query that has waited
``threshold`` (sim.py:297-332, 477-478; prefetch.py:63-72).  This module runs
the same policy for real, on the wall clock, one process per GPU:

* **Instances** (:class:`Instance`, one per GPU/process) each run a *serve
  thread* that pulls batches from the node-wide FIFO (``control.ControlPlane``,
  shared memory) whenever idle, and a *generator thread* that serves the
  instance's generation-request ring on a low-priority CUDA stream, so
  precompute overlaps serving on the same GPU.
* **Precompute is owner-partitioned**: the request for a query's combination
  goes to ``owner_rank(KvKey(combination))``; the owner claims each missing
  prefix key through the control plane's cross-process single-flight state,
  runs ONE row-deterministic prefill of the combination and derives every
  prefix from it (SURVEY H-e, bit-identical to from-scratch prefixes), places
  the KV in its HBM tier (prefixes share the combination's pool blocks),
  publishes the residency, and persists the blobs to the shared store
  (``persist`` policy) on a writer thread.
* **Lookup order** for each prefix (longest first): this GPU's HBM tier,
  a peer's HBM tier (pulled over NVLink by K3p while the holder's entry is
  pinned in the control plane), then the shared ``KvStore`` (memory tier, then
  disk: the reference's tiers, with their accounting), else a miss that
  prefills raw text (costs.py:136-138).
* **Queue monitor** (rank 0, :class:`Driver`): replays the arrival schedule on
  the wall clock, pushes queries into the FIFO and calls ``prefetch.scan`` at
  the threshold for queries not yet dispatched.

TTFT is measured as the reference defines it (kv_load + prefill, here the
dispatch-to-first-token wall time) and arrival-to-first-token.
"""

from __future__ import annotations

import os
import queue
import threading
import time
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from .control import ControlPlane, Counter, KeyState, QState
from .engine import Engine
from .generator import KvGenerator
from .model import combo_tokens, query_tokens
from .multi import owner_rank
from .prefetch import PendingQuery, scan
from . import decode
from .prefill import PrefillRequest, prefill_batch
from .store import CacheTier, KvKey, KvStore, LookupResult, Outcome

STOP = 31  # control-plane counter: serving threads exit when it is non-zero


@dataclass
class RuntimeConfig:
    k: int                              # documents per query (SimConfig.k)
    threshold: float = 0.5              # queue wait before a query is flagged (paper.json:83)
    prefetch: bool = True               # queue-time proactive precompute on
    max_batch: int = 16                 # queries an idle instance takes from the FIFO at once
    max_batch_tokens: int = 16384       # new tokens per serving batch (>= one query always)
    persist: str = "all"                # generated blobs put in the store: "all" prefixes | "composite" | "none"
    token_seed: int = 0
    idle_sleep_s: float = 2e-4
    # Cost-aware dispatch (opt-in deviation from the reference's "longest cached prefix
    # wins", sim.py:414-431): a prefix found only on DISK is used only if reading it is
    # predicted faster than recomputing its tokens; otherwise the next-best non-disk
    # prefix (or raw prefill) is served and the disk copy is left alone.  On a B200 an
    # 8B composite of 5120 tokens reads in ~190 ms from a ~3.4 GB/s disk but prefills in
    # ~55 ms (bench ttft_ms.cold_disk vs full_prefill), so the reference rule loses there.
    cost_aware: bool = False
    disk_gbps: float = 5.0              # cold O_DIRECT read of the shared store (scripts/micro/cold_path.py)
    prefill_s_per_token: float = 1.1e-5 # measured full-prefill cost per prefix token on this GPU
    # Decode after the first token (decode.py; the reference's decode_tokens, sim.py:572-573):
    # every query generates this many more tokens greedily; the instance batches them
    # continuously (new queries' prefills join between decode steps, finished ones leave).
    # A query is DONE when its last token is out; TTFT stays the first token's.
    decode_tokens: int = 0
    # Chunked prefill (with decode_tokens > 0): at most this many prompt tokens per forward,
    # shared first-come-first-served by the prompts still being prefilled, each forward also
    # carrying one decode token per running query (decode.extend) — a long miss prefill no longer
    # stalls every decoding query for its whole duration (TPOT) at the cost of the chunked
    # prompts' own TTFT.  0 = whole prompts at once.
    prefill_chunk: int = 0

    def __post_init__(self) -> None:
        if self.persist not in ("all", "composite", "none"):
            raise ValueError("persist must be 'all', 'composite' or 'none'")


@dataclass
class QueryResult:
    index: int
    query_id: int
    rank: int
    arrival: float              # monotonic seconds
    dispatch: float
    first_token: float
    best: int                   # cached prefix length used (documents)
    source: str                 # where that prefix came from: hbm | peer | memory | disk | miss
    origins: tuple              # per prefix j: generated | hbm | peer | memory | disk | miss_raw
    batch: int                  # queries in the serving batch
    token: int                  # first token
    done: float = 0.0           # last token out (decode_tokens > 0; = first_token otherwise)
    n_tokens: int = 1           # tokens generated, the first one included
    tokens: tuple = ()          # every generated token (decode_tokens > 0)

    @property
    def latency(self) -> float:
        return self.first_token - self.arrival

    @property
    def ttft(self) -> float:    # reference definition: kv_load + prefill (sim.py:450-454), no queueing
        return self.first_token - self.dispatch


@dataclass
class AccessRecord:
    """One access that reached the shared store (SURVEY H-i replay unit)."""
    key: tuple
    outcome: str
    load_cost_bytes: int


class _Writer:
    """Write-behind persistence of generated blobs into the shared store."""

    def __init__(self, store: KvStore, cp: ControlPlane, depth: int = 8) -> None:
        self.store, self.cp = store, cp
        self.q: "queue.Queue" = queue.Queue(maxsize=depth)
        self.errors: list = []
        self.th = threading.Thread(target=self._run, name="rdkv-writer", daemon=True)
        self.th.start()

    def _run(self) -> None:
        while True:
            item = self.q.get()
            if item is None:
                return
            key, blob = item
            try:
                self.store.put(key, blob)
                self.cp.add(Counter.STORE_PUTS)
            except Exception as exc:  # surfaced by Instance.close
                self.errors.append((key, exc))
            finally:
                self.q.task_done()

    def submit(self, key: KvKey, blob) -> None:
        self.q.put((key, blob))

    def drain(self) -> None:
        self.q.join()

    def close(self) -> None:
        self.q.put(None)
        self.th.join(timeout=60)


class Instance:
    """One model instance (one GPU, one process) of the serving runtime."""

    def __init__(self, engine: Engine, store: KvStore, cp: ControlPlane, cfg: RuntimeConfig,
                 peers=None) -> None:
        self.eng, self.store, self.cp, self.cfg = engine, store, cp, cfg
        self.rank, self.world = cp.rank, cp.world
        self.peers = peers                      # multi.PeerPools (CUDA IPC maps of every rank's pool) or None
        self.profile = engine.spec.profile()
        self.mh = self.profile.model_hash
        lo, hi = torch.cuda.Stream.priority_range() if torch.cuda.is_available() else (0, 0)
        # serving gets the highest priority; queue-time generation the lowest
        self.serve_stream = torch.cuda.Stream(device=engine.device, priority=hi)
        self.gen_stream = torch.cuda.Stream(device=engine.device, priority=lo)
        engine.pool.reader_stream = self.serve_stream
        engine.resident.can_evict = self._can_evict
        self.gen = KvGenerator(engine, token_seed=cfg.token_seed, keep_on_device=False)
        self.gen.copy_stream = torch.cuda.Stream(device=engine.device, priority=lo)
        self.results: list[QueryResult] = []
        self.access_log: list[AccessRecord] = []
        self.generated: list[tuple[int, tuple]] = []     # (requesting query index, prefix ids) per key made here
        self._gen_for: dict[tuple, int] = {}             # prefix ids -> query index that triggered it
        self._unpins: list = []                           # (event, key): peer pins to drop once copies land
        self._live: list = []                             # (decode.DecodeSeq, result index) being decoded
        self._filling: list = []                          # [LiveSequence, remaining tokens, meta, t_dispatch, batch]
        self._writer = _Writer(store, cp)
        self._threads: list[threading.Thread] = []
        self.errors: list = []

    # ------------------------------------------------------------ lifecycle
    def warmup(self) -> None:
        """First launches on each stream set kernel attributes and allocate the
        per-stream workspaces: do them before the clock starts."""
        spec = self.eng.spec
        toks = np.arange(64, dtype=np.int32) % spec.vocab
        with torch.cuda.stream(self.gen_stream):
            self.eng.generate_doc_kv(toks, stream=self.gen_stream)
        with torch.cuda.stream(self.serve_stream):
            prefill_batch(self.eng, [PrefillRequest(LookupResult(Outcome.MISS), toks[:32], toks[32:])],
                          timed=False, use_graph=False)
        torch.cuda.synchronize(self.eng.device)

    def start(self) -> None:
        for name, fn in (("serve", self._serve_loop), ("generate", self._gen_loop)):
            th = threading.Thread(target=self._guard(fn), name=f"rdkv-{name}-{self.rank}", daemon=True)
            th.start()
            self._threads.append(th)

    def _guard(self, fn):
        def run():
            try:
                torch.cuda.set_device(self.eng.device)
                fn()
            except BaseException as exc:  # a crashed worker stops the node instead of hanging it
                self.errors.append(exc)
                self.cp.add(STOP)
                raise
            finally:
                if os.environ.get("RDKV_RT_DEBUG"):
                    import sys
                    print(f"[rdkv runtime] rank {self.rank} {threading.current_thread().name} exits "
                          f"(stop={self.cp.counter(STOP)}, errors={self.errors!r})", file=sys.stderr, flush=True)
        return run

    def join(self) -> None:
        for th in self._threads:
            th.join()
        self._threads = []
        self._writer.drain()
        self._drain_unpins(block=True)

    def close(self) -> None:
        self._writer.close()
        if self._writer.errors:
            raise RuntimeError(f"store writes failed: {self._writer.errors[:2]}")

    def stopping(self) -> bool:
        return self.cp.counter(STOP) != 0

    # ------------------------------------------------------------ residency
    def _can_evict(self, key) -> bool:
        return not isinstance(key, KvKey) or self.cp.retract(key)

    def _drain_unpins(self, block: bool = False) -> None:
        keep = []
        for ev, key in self._unpins:
            if block:
                ev.synchronize()
            if ev.query():
                self.cp.unpin(key)
            else:
                keep.append((ev, key))
        self._unpins = keep

    def _source(self, key: KvKey) -> str | None:
        if key in self.eng.resident:
            return "hbm"
        h = self.cp.holder(key)
        if h is not None and h != self.rank and self.peers is not None:
            return "peer"
        tier = self.store.contains(key)
        if tier is CacheTier.ABSENT and self.cp.key_state(key)[0] is KeyState.READY:
            self.store.refresh()  # another instance's put landed in the shared manifest
            tier = self.store.contains(key)
        if tier is CacheTier.IN_MEMORY:
            return "memory"
        if tier is CacheTier.ON_DISK:
            return "disk"
        return None

    def _peer_fetch(self, key: KvKey) -> bool:
        """Pull ``key``'s KV from the peer holding it in HBM (K3p over NVLink) into
        this GPU's HBM tier; the holder cannot evict it while our pin is held."""
        got = self.cp.pin(key)
        if got is None:
            return False
        holder, blocks, n = got
        if holder == self.rank:
            self.cp.unpin(key)
            return False
        dst = self.eng.resident.reserve(n)
        if dst is None:
            self.cp.unpin(key)
            return False
        self.peers.gather(holder, blocks[: len(dst)], dst, stream=self.serve_stream)
        ev = torch.cuda.Event()
        ev.record(self.serve_stream)
        self.eng.resident.commit(key, dst, n, ready=ev)
        self._unpins.append((ev, key))
        self.cp.add(Counter.PEER_FETCHES)
        self.cp.add(Counter.PEER_BYTES, n * self.eng.spec.kv_bytes_per_token())
        return True

    # ------------------------------------------------------------ serving
    def _serve_loop(self) -> None:
        with torch.cuda.stream(self.serve_stream):
            try:
                while not self.stopping():
                    self._drain_unpins()
                    room = self.cfg.max_batch - len(self._live) - len(self._filling)
                    batch = self._take_batch(room) if room > 0 else []
                    if batch:
                        self._serve(batch)
                    if self._filling:
                        self._mixed_step()
                    elif self._live:
                        self._decode_step()
                    elif not batch:
                        time.sleep(self.cfg.idle_sleep_s)
            finally:
                for seq, _ in self._live:
                    decode.retire(self.eng, seq)
                for lv, *_ in self._filling:
                    decode.retire(self.eng, decode.DecodeSeq(lv, 0, 1))
                self._live = []
                self._filling = []

    def _mixed_step(self) -> None:
        """One forward: a decode token for every live sequence plus the next chunk of every
        prompt being prefilled in chunks; a prompt whose last chunk ran yields its first token
        (TTFT) and starts decoding."""
        cfg = self.cfg
        dec = [(s, ri) for s, ri in self._live if not s.done]
        parts = [(s.live, np.array([s.last], np.int32)) for s, _ in dec]
        budget = cfg.prefill_chunk
        fed = []
        for f in self._filling:  # first come, first served
            if budget <= 0:
                break
            chunk, f[1] = f[1][:budget], f[1][budget:]
            budget -= len(chunk)
            fed.append(f)
            parts.append((f[0], chunk))
        nxt = decode.extend(self.eng, parts).cpu().tolist() if parts else []
        now = time.monotonic()
        for (s, _), t in zip(dec, nxt[: len(dec)]):
            s.last = int(t)
            s.tokens.append(int(t))
        done = set()
        for f, t in zip(fed, nxt[len(dec):]):
            lv, rest, meta, t_dispatch, nb = f
            if not len(rest):
                self._first_token(lv, int(t), meta, t_dispatch, now, nb)
                done.add(id(f))
        self._filling = [f for f in self._filling if id(f) not in done]
        self._retire_done(now)

    def _first_token(self, lv, tok: int, meta, t_dispatch: float, t_first: float, batch_n: int) -> None:
        index, qid, arrival, best, source, origins = meta
        self.results.append(QueryResult(index, qid, self.rank, arrival, t_dispatch, t_first, best, source,
                                        origins, batch_n, tok, t_first))
        self._live.append((decode.DecodeSeq(lv, tok, self.cfg.decode_tokens + 1, [tok]), len(self.results) - 1))

    def _retire_done(self, now: float) -> None:
        keep = []
        for seq, ri in self._live:
            if seq.done:
                res = self.results[ri]
                res.done, res.n_tokens, res.tokens = now, len(seq.tokens), tuple(seq.tokens)
                decode.retire(self.eng, seq)
                self.cp.qstate_cas(res.index, QState.DISPATCHED, QState.DONE)
            else:
                keep.append((seq, ri))
        self._live = keep

    def _decode_step(self) -> None:
        """One decode step for every live sequence (continuous batching); finished
        sequences leave the batch, their queries become DONE."""
        decode.step(self.eng, [s for s, _ in self._live])
        self._retire_done(time.monotonic())

    def _take_batch(self, limit: int | None = None) -> list:
        """An idle instance takes the oldest waiting queries (up to max_batch /
        max_batch_tokens new tokens; the reference dispatches one query per idle
        instance, sim.py:403-409 — batching only groups what already waits)."""
        out, tokens = [], 0
        limit = self.cfg.max_batch if limit is None else limit
        while len(out) < limit:
            q = self.cp.pop_query()
            if q is None:
                break
            index = q[0]
            if not self.cp.qstate_cas(index, QState.QUEUED, QState.DISPATCHED):
                raise RuntimeError(f"query {index} popped twice")
            out.append(q)
            tokens += sum(q[5][: self.cfg.k]) + q[3]
            if tokens >= self.cfg.max_batch_tokens:
                break
        return out

    def _serve(self, batch) -> None:
        cfg, spec = self.cfg, self.eng.spec
        t_dispatch = time.monotonic()
        reqs, meta = [], []
        for index, qid, arrival, qn, ids, counts in batch:
            combo, toks = tuple(ids[: cfg.k]), tuple(counts[: cfg.k])
            keys = [KvKey(self.mh, combo[:j]) for j in range(1, len(combo) + 1)]
            srcs = [self._source(key) for key in keys]
            best = max((j for j, s in enumerate(srcs, 1) if s is not None), default=0)
            source = srcs[best - 1] if best else "miss"
            if cfg.cost_aware and source == "disk" and self._disk_loses(sum(toks[:best])):
                self.cp.add(Counter.DISK_SKIPPED)
                best = max((j for j, s in enumerate(srcs[: best - 1], 1) if s in ("hbm", "peer", "memory")),
                           default=0)
                source = srcs[best - 1] if best else "miss"
            q = query_tokens(qid, qn, spec.vocab, cfg.token_seed)
            if source == "peer" and not self._peer_fetch(keys[best - 1]):
                # the holder evicted it meanwhile: next-best source for the same prefix
                self.store.refresh()
                tier = self.store.contains(keys[best - 1])
                source = {CacheTier.IN_MEMORY: "memory", CacheTier.ON_DISK: "disk"}.get(tier)
                if source is None:
                    best = max((j for j, s in enumerate(srcs[: best - 1], 1) if s in ("hbm", "memory", "disk")),
                               default=0)
                    source = srcs[best - 1] if best else "miss"
            rest = combo_tokens(combo[best:], toks[best:], spec.vocab, cfg.token_seed)
            new = np.concatenate([rest, q]) if len(rest) else q
            if source in ("hbm", "peer"):
                req = PrefillRequest(LookupResult(Outcome.MEMORY_HIT, None, 0), None, new, keys[best - 1])
            elif source in ("memory", "disk"):
                look = self.store.get(keys[best - 1])          # the reference tiers, real I/O and accounting
                self.access_log.append(AccessRecord(keys[best - 1].doc_ids, look.outcome.value, look.load_cost_bytes))
                if look.outcome is Outcome.MISS:
                    raise RuntimeError(f"store lost {keys[best - 1]}")
                req = PrefillRequest(look, None, new, None)
            else:
                req = PrefillRequest(LookupResult(Outcome.MISS), combo_tokens(combo, toks, spec.vocab,
                                                                              cfg.token_seed), q)
            origins = tuple("generated" if s is not None and self._gen_for.get(combo[:j]) == index
                            else ("miss_raw" if s is None else s) for j, s in enumerate(srcs, 1))
            reqs.append(req)
            meta.append((index, qid, arrival, best, source, origins))
        dec = cfg.decode_tokens > 0
        rests = [np.zeros(0, np.int32)] * len(reqs)
        if dec and cfg.prefill_chunk > 0:  # chunked prefill: a share of the budget now, the rest in mixed steps
            share = max(1, cfg.prefill_chunk // len(reqs))
            for i, req in enumerate(reqs):
                whole = np.asarray(req.new_tokens, np.int32) if req.lookup.outcome is not Outcome.MISS else \
                    np.concatenate([np.asarray(req.prefix_tokens, np.int32), np.asarray(req.new_tokens, np.int32)])
                if len(whole) > share:
                    head, rests[i] = whole[:share], whole[share:]
                    reqs[i] = PrefillRequest(req.lookup, head[:0], head, req.key) \
                        if req.lookup.outcome is not Outcome.MISS else PrefillRequest(req.lookup, head, head[:0], None)
        r = prefill_batch(self.eng, reqs, timed=False, use_graph=False, keep=dec)
        first = r.next_token.cpu()  # D2H of the first tokens: the batch's TTFT point
        t_first = time.monotonic()
        if any(len(x) for x in rests):
            keep_meta, keep_first = [], []
            for i, m in enumerate(meta):
                if len(rests[i]):
                    self._filling.append([r.sequences[i], rests[i], m, t_dispatch, len(batch)])
                else:
                    keep_meta.append((i, m))
            for i, m in keep_meta:
                self._first_token(r.sequences[i], int(first[i]), m, t_dispatch, t_first, len(batch))
            return
        for i, ((index, qid, arrival, best, source, origins), tok) in enumerate(zip(meta, first.tolist())):
            self.results.append(QueryResult(index, qid, self.rank, arrival, t_dispatch, t_first, best, source,
                                            origins, len(batch), int(tok), t_first))
            if dec:  # keeps its KV: decoded by the next steps, DONE with its last token
                self._live.append((decode.DecodeSeq(r.sequences[i], int(tok), cfg.decode_tokens + 1, [int(tok)]),
                                   len(self.results) - 1))
            else:
                self.cp.qstate_cas(index, QState.DISPATCHED, QState.DONE)

    def _disk_loses(self, n_tokens: int) -> bool:
        """Cost-aware dispatch: is reading ``n_tokens`` of cached KV from disk predicted
        slower than prefilling them (kv_load vs prefill terms of costs.py:125-144)?"""
        load = n_tokens * self.eng.spec.kv_bytes_per_token() / (self.cfg.disk_gbps * 1e9)
        return load > n_tokens * self.cfg.prefill_s_per_token

    # ------------------------------------------------------------ queue-time generation
    def _gen_loop(self) -> None:
        with torch.cuda.stream(self.gen_stream):
            while not self.stopping():
                req = self.cp.pop_request()
                if req is None:
                    time.sleep(self.cfg.idle_sleep_s)
                    continue
                index, ids, counts = req
                try:
                    self._generate(index, tuple(ids), tuple(counts))
                except Exception as exc:  # best effort (prefetch.py:129-157): failures free the keys
                    self.errors.append(exc)
                    self.cp.add(Counter.GENERATION_FAILURES)

    def _generate(self, index: int, ids: tuple, counts: tuple) -> None:
        cp, eng = self.cp, self.eng
        keys = [KvKey(self.mh, ids[:j]) for j in range(1, len(ids) + 1)]
        claimed = claim_keys(cp, keys)
        if not claimed:
            return
        try:
            jmax = max(claimed)
            ntok = [sum(counts[:j]) for j in range(len(ids) + 1)]
            toks = combo_tokens(ids[:jmax], counts[:jmax], eng.spec.vocab, self.cfg.token_seed)
            kv = eng.generate_doc_kv(toks, stream=self.gen_stream)      # one row-deterministic prefill
            cp.add(Counter.GENERATION_RUNS)
            base = keys[jmax - 1]
            resident = eng.make_resident(base, kv, ntok[jmax], stream=self.gen_stream)
            if resident:
                for j in claimed:
                    if j != jmax:
                        eng.resident.alias(keys[j - 1], base, ntok[j])
                ready = eng.resident.get(base).ready
                if ready is not None:
                    ready.synchronize()                                  # blocks written before peers see them
                for j in claimed:
                    e = eng.resident.get(keys[j - 1])
                    if e is not None:
                        cp.publish(keys[j - 1], e.blocks, e.n_tokens)
            persist = {"all": claimed, "composite": [jmax], "none": []}[self.cfg.persist]
            if not resident:
                persist = claimed  # no HBM room: the store is the only place it can live
            for j in persist:
                payload = self.gen.slice_prefix(kv, ntok[jmax], ntok[j])
                blob = self.gen._blob_from_device(ids[:j], ntok[j], payload)   # GPU FNV-1a + D2H
                # write-behind: the key is already served from HBM; the bounded writer
                # queue throttles generation when the disk falls behind
                self._writer.submit(keys[j - 1], blob)
            if not resident and persist:
                self._writer.drain()  # nowhere else to read it from until the put lands
        except BaseException:
            for j in claimed:
                cp.key_cas(keys[j - 1], KeyState.GENERATING, KeyState.FAILED)
            raise
        for j in claimed:
            self._gen_for[ids[:j]] = index
            self.generated.append((index, ids[:j]))
        finish_keys(cp, [keys[j - 1] for j in claimed])


def claim_keys(cp: ControlPlane, keys: Sequence[KvKey]) -> list[int]:
    """Cross-process single flight (service.py:87-127): claim every key not yet
    being generated or made; returns the 1-based prefix lengths this rank won."""
    won = []
    for j, key in enumerate(keys, 1):
        if any(cp.key_cas(key, s, KeyState.GENERATING) for s in (KeyState.REQUESTED, KeyState.ABSENT,
                                                                   KeyState.FAILED)):
            won.append(j)
        else:
            cp.add(Counter.CLAIMS_LOST)
    return won


def finish_keys(cp: ControlPlane, keys: Sequence[KvKey]) -> None:
    for key in keys:
        if not cp.key_cas(key, KeyState.GENERATING, KeyState.READY):
            raise RuntimeError(f"{key} was not GENERATING by this rank")
        cp.add(Counter.KEYS_GENERATED)
        cp.add(Counter.PER_RANK_GENERATED + cp.rank)


class Driver:
    """Rank 0's arrival replay and queue monitor (sim.py:462-478, prefetch.scan)."""

    def __init__(self, cp: ControlPlane, cfg: RuntimeConfig, model_hash: int, store: KvStore | None = None) -> None:
        self.cp, self.cfg, self.mh, self.store = cp, cfg, model_hash, store
        self.flagged = 0
        self.requests = 0

    def _present(self, key: KvKey) -> bool:
        st, _ = self.cp.key_state(key)
        if st in (KeyState.READY, KeyState.GENERATING, KeyState.REQUESTED):
            return True
        return self.cp.holder(key) is not None or (self.store is not None and
                                                   self.store.contains(key) is not CacheTier.ABSENT)

    def _flag(self, pq: PendingQuery) -> None:
        """plan_tasks (prefetch.py:104-126): every missing prefix; the owner of the
        combination generates all of them from one prefill."""
        combo, counts = tuple(pq.doc_ids[: self.cfg.k]), tuple(pq.doc_tokens[: self.cfg.k])
        missing = False
        for j in range(1, len(combo) + 1):
            key = KvKey(self.mh, combo[:j])
            if self._present(key):
                continue
            if self.cp.key_cas(key, KeyState.ABSENT, KeyState.REQUESTED) or \
                    self.cp.key_cas(key, KeyState.FAILED, KeyState.REQUESTED):
                missing = True
        if missing:
            owner = owner_rank(KvKey(self.mh, combo), self.cp.world)
            while not self.cp.push_request(owner, combo, counts, pq.query_id):
                time.sleep(1e-4)
            self.cp.add(Counter.GENERATION_REQUESTS)
            self.requests += 1

    def run(self, arrivals: Sequence[tuple[float, object]], index0: int, t0: float,
            deadline_s: float = 900.0) -> None:
        """Push ``arrivals`` ((offset seconds, WorkItem), sorted) at t0 + offset;
        flag waiting queries at the threshold; return when all are served
        (raise if that takes longer than ``deadline_s``)."""
        cfg = self.cfg
        deadline = t0 + deadline_s
        pending: list[PendingQuery] = []
        n, i = len(arrivals), 0
        while True:
            now = time.monotonic()
            while i < n and t0 + arrivals[i][0] <= now:
                off, it = arrivals[i]
                index = index0 + i
                self.cp.qstate_cas(index, QState.NONE, QState.QUEUED)
                while not self.cp.push_query(index, it.query_id, t0 + off, it.q_tokens, it.doc_ids[: cfg.k],
                                             it.doc_tokens[: cfg.k]):
                    time.sleep(1e-4)
                if cfg.prefetch:
                    pending.append(PendingQuery(index, t0 + off, cfg.k, it.q_tokens, tuple(it.doc_ids),
                                                tuple(it.doc_tokens)))
                i += 1
            if pending:
                pending = [p for p in pending if self.cp.qstate(p.query_id) is QState.QUEUED]
                for qi in scan(pending, now, cfg.threshold):
                    self.flagged += 1
                    self._flag(next(p for p in pending if p.query_id == qi))
            if i == n and all(self.cp.qstate(index0 + j) is QState.DONE for j in range(n)):
                return
            if self.cp.counter(STOP):
                raise RuntimeError("an instance stopped the node (worker error)")
            if now > deadline:
                raise TimeoutError(f"{sum(self.cp.qstate(index0 + j) is not QState.DONE for j in range(n))} of "
                                   f"{n} queries unserved after {deadline_s:.0f} s")
            nxt = [t0 + arrivals[i][0]] if i < n else []
            nxt += [p.arrival_time + cfg.threshold for p in pending if not p.flagged]
            wait = (min(nxt) - time.monotonic()) if nxt else cfg.idle_sleep_s
            time.sleep(min(max(wait, 0.0), 1e-3) if wait > 0 else 0.0)


def summarize(results: Sequence[QueryResult], tries: Sequence[Sequence[QueryResult]] | None = None) -> dict:
    """TTFT percentiles (both definitions) and throughput.  Throughput divides by
    the SUM of per-try makespans (reference build_report, sim.py:226-240), never
    by one span across tries."""
    lat = np.array([r.latency for r in results])
    ttft = np.array([r.ttft for r in results])
    groups = tries if tries is not None else [results]
    # a try ends with its last token out (the first token unless queries decode: the reference
    # adds decode time to the batch span, sim.py:572-573)
    spans = [max(max(r.first_token, r.done) for r in g) - min(r.arrival for r in g) for g in groups if g]
    origins: dict[str, int] = {}
    sources: dict[str, int] = {}
    for r in results:
        sources[r.source] = sources.get(r.source, 0) + 1
        for o in r.origins:
            origins[o] = origins.get(o, 0) + 1
    pct = lambda a: {"p50": float(np.percentile(a, 50) * 1e3), "p99": float(np.percentile(a, 99) * 1e3)}
    return {
        "queries": len(results),
        "qps": len(results) / sum(spans) if spans and sum(spans) > 0 else 0.0,
        "per_try_qps": [len(g) / s for g, s in zip([g for g in groups if g], spans)],
        "latency_ms": pct(lat), "ttft_ms": pct(ttft),
        "mean_batch": float(np.mean([r.batch for r in results])),
        "sources": dict(sorted(sources.items())), "origins": dict(sorted(origins.items())),
        **_decode_summary(results, spans),
    }


def _decode_summary(results: Sequence[QueryResult], spans) -> dict:
    dec = [r for r in results if r.n_tokens > 1]
    if not dec:
        return {}
    tpot = np.array([(r.done - r.first_token) / (r.n_tokens - 1) for r in dec])
    toks = sum(r.n_tokens for r in results)
    return {"decode": {"queries": len(dec), "tokens": int(toks),
                       "tokens_per_s": toks / sum(spans) if sum(spans) > 0 else 0.0,
                       "tpot_ms": {"p50": float(np.percentile(tpot, 50) * 1e3),
                                   "p99": float(np.percentile(tpot, 99) * 1e3)}}}


def arrivals_for_try(items: Sequence, rate: float, seed: int, try_index: int) -> list[tuple[float, object]]:
    """The reference's per-try arrival schedule (sim.py:340-355): the same Poisson
    timestamps every try, a freshly seeded item order."""
    from .workload import poissonize

    perm = np.random.default_rng([seed, try_index, 0x5EED]).permutation(len(items))
    order = [items[i] for i in perm]
    arrival_seed = int(np.random.default_rng([seed, 0xA221]).integers(0, 2 ** 63))
    return poissonize(order, rate, seed=arrival_seed)


def serve(engine: Engine, store: KvStore, cfg: RuntimeConfig, items: Sequence, rate: float, tries: int = 1,
          seed: int = 1, rank: int = 0, world: int = 1, peers=None, group=None) -> dict | None:
    """Serve ``items`` (WorkItems with doc ids) arriving as a Poisson process of
    ``rate`` q/s, ``tries`` passes with the cache carried over (sim.py:343-355),
    on this node's ``world`` instances.  Call on every rank; rank 0 drives the
    arrivals and returns the report (None elsewhere)."""
    dist = None
    if world > 1:
        import torch.distributed as dist
    names = [f"/rdkv_rt_{os.getpid()}_{time.monotonic_ns() % 10**9}"]
    if dist is not None:
        dist.broadcast_object_list(names, src=0, group=group)
    cp = ControlPlane(names[0], rank, world, create=rank == 0)
    if dist is not None:
        dist.barrier(group=group)
    inst = Instance(engine, store, cp, cfg, peers)
    inst.warmup()
    if dist is not None:
        dist.barrier(group=group)
    inst.start()
    out = None
    try:
        if rank == 0:
            driver = Driver(cp, cfg, inst.mh, store)
            wall = []
            for t in range(tries):
                arr = arrivals_for_try(items, rate, seed, t + 1)
                t0 = time.monotonic() + 0.002
                driver.run(arr, t * len(items), t0)
                wall.append(time.monotonic() - t0)
            cp.add(STOP)
    except BaseException:
        cp.add(STOP)
        raise
    finally:
        inst.join()
    results = inst.results
    generated = inst.generated
    access = inst.access_log
    if dist is not None:
        allr, allg = [None] * world, [None] * world
        dist.all_gather_object(allr, results, group=group)
        dist.all_gather_object(allg, generated, group=group)
        results = [r for lst in allr for r in lst]
        generated = [g for lst in allg for g in lst]
        dist.barrier(group=group)
    if inst.errors:
        raise RuntimeError(f"rank {rank}: runtime worker failed: {inst.errors[0]!r}") from inst.errors[0]
    if rank == 0:
        n = len(items)
        per_try = [[r for r in results if r.index // n == t] for t in range(tries)]
        rep = summarize(results, per_try)
        keys = [g[1] for g in generated]
        counters = cp.counters()
        rep.update({
            "rate": rate, "tries": tries, "instances": world, "wall_s_per_try": wall,
            "flagged": driver.flagged, "generation_requests": driver.requests,
            "keys_generated": len(keys), "distinct_keys_generated": len(set(keys)),
            "each_key_generated_once": len(keys) == len(set(keys)) == counters["keys_generated"],
            "counters": counters, "store_accesses_rank0": len(access),
            "hbm_tier": {"entries": len(engine.resident), "blocks": engine.resident.used,
                         "evictions": engine.resident.evictions},
        })
        out = {"summary": rep, "results": results, "access_log": access, "generated": generated}
    inst.close()
    if dist is not None:
        dist.barrier(group=group)
    cp.close(unlink=rank == 0)
    return out
