"""Serving on B200: the reference scheduling policy driven by real GPU work.

``sim.run`` (the reference policy, sim.py:358-504) asks an executor how long
each dispatch and each queue-time generation takes.  :class:`MeasuredExecutor`
answers by *doing* the work on a B200 and timing it:

* a dispatch looks the longest cached prefix up in the real
  :class:`~paper_2504_11765_b200.store.KvStore` (MEMORY_HIT: pinned host payload;
  DISK_HIT: aligned read + FNV verify), copies the payload to HBM, unpacks it
  into the paged pool (K3) and prefills the remaining documents + query over it
  (K1/K2/K4/K5) — ``kv_load`` is host lookup + H2D + unpack, ``prefill`` the
  forward, both measured;
* a miss prefills the whole prompt from raw tokens (costs.py:136-138);
* a queue-time generation runs the document prefill of the prefix combination,
  hashes it and ``put``s it through the single-flight service
  (sim.py:319-332 / prefetch.py:129-157) — its measured wall time is the
  generator busy time.

The policy's cache mirror (``TierMirror``) and the real store see the same
inserts and promotions, so the decision sequence stays identical to the
reference's; every real store outcome is logged (``access_log``) and checked
against the mirror's tier (SURVEY H-i: replaying the log into the reference
store reproduces outcomes and stats).  Run with ``memory_capacity_bytes = 0``
(the paper's shared-experiment setting) or equal capacities on both sides.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .costs import Tier
from .engine import Engine
from .generator import KvGenerator
from .model import combo_tokens, query_tokens
from .prefill import PrefillRequest, prefill_batch
from .service import SharedCacheService
from .sim import Dispatch, GenTask, SimConfig, TierMirror
from .store import KvKey, LookupResult, Outcome


@dataclass
class AccessRecord:
    query_id: int
    prefix: tuple[int, ...]
    mirror_tier: str          # "memory" | "disk" | "miss"
    outcome: str              # real store outcome
    kv_load_s: float
    prefill_s: float
    first_token: int


@dataclass
class MeasuredExecutor:
    """Executor for ``sim.run`` that executes every decision on the GPU."""

    engine: Engine
    service: SharedCacheService
    token_seed: int = 0
    access_log: list[AccessRecord] = field(default_factory=list)
    generations: list[tuple[tuple[int, ...], float]] = field(default_factory=list)
    # query_id -> WorkItem: lets a generation task find its waiting query's whole
    # combination and run one prefill for all of that combination's prefixes
    workload: dict | None = None
    _combos: "OrderedDict" = field(default_factory=lambda: __import__("collections").OrderedDict())

    def bind(self, config: SimConfig, cache: TierMirror) -> None:
        self.cfg = config
        self.cache = cache
        self.gen = KvGenerator(self.engine, token_seed=self.token_seed, keep_on_device=False)
        self.profile = self.engine.spec.profile()
        if config.memory_capacity_bytes != self.service.store.stats().memory_capacity_bytes:
            raise ValueError("store memory capacity must equal the simulated one (lock-step tiers)")

    def _tokens(self, ids, counts) -> np.ndarray:
        return combo_tokens(ids, counts, self.engine.spec.vocab, self.token_seed)

    def serve(self, d: Dispatch) -> tuple[float, float]:
        vocab = self.engine.spec.vocab
        q = query_tokens(d.item.query_id, d.item.q_tokens, vocab, self.token_seed)
        torch.cuda.synchronize(self.engine.device)
        t0 = time.perf_counter()
        if d.best > 0:
            prefix = tuple(d.combo[: d.best])
            look = self.service.get(KvKey(self.profile.model_hash, prefix))  # real tier, real I/O
            if look.outcome is Outcome.MISS:
                raise RuntimeError(f"store lost {prefix} that the policy mirror holds")
            rest = self._tokens(d.combo[d.best:], d.tokens[d.best:])
            new = np.concatenate([rest, q]) if len(rest) else q
            req = PrefillRequest(look, None, new)
            mirror = "memory" if d.tier is Tier.MEMORY else "disk"
        else:
            look = LookupResult(Outcome.MISS)
            req = PrefillRequest(look, self._tokens(d.combo, d.tokens), q)
            prefix, mirror = (), "miss"
        host_s = time.perf_counter() - t0
        r = prefill_batch(self.engine, [req], timed=True)
        first = int(r.next_token[0])
        kv_load = host_s + r.breakdown.kv_load
        self.access_log.append(AccessRecord(d.item.query_id, prefix, mirror, look.outcome.value, kv_load,
                                            r.breakdown.prefill, first))
        return kv_load, r.breakdown.prefill

    def _factory(self, ids, counts):
        """Per-prefix generate factory; shares one combination prefill when a waiting
        query's combination extends this prefix (KvGenerator.for_combination)."""
        if self.workload:
            for combo, fac in self._combos.items():
                if combo[: len(ids)] == ids:
                    return fac
            return None
        return None

    def generation_time(self, task: GenTask) -> float:
        ids = task.prefix
        counts = self._doc_counts(ids, task.span_tokens)
        key = KvKey(self.profile.model_hash, ids)
        t0 = time.perf_counter()
        fac = self._factory(ids, counts)
        if fac is None and self.workload:
            for q in sorted(task.waiters):
                it = self.workload.get(q)
                if it is not None and tuple(it.doc_ids[: self.cfg.k])[: len(ids)] == ids:
                    combo = tuple(it.doc_ids[: self.cfg.k])
                    fac = self.gen.for_combination(combo, tuple(it.doc_tokens[: self.cfg.k]))
                    self._combos[combo] = fac
                    while len(self._combos) > 4:  # each holds one combination's KV in HBM
                        self._combos.popitem(last=False)
                    break
        self.service.get_or_generate(key, (fac or self.gen.for_prefix)(ids, counts))
        dt = time.perf_counter() - t0
        self.generations.append((ids, dt))
        return dt

    def generated(self, task: GenTask) -> None:
        pass

    def _doc_counts(self, ids, span: int) -> tuple[int, ...]:
        # workloads give every doc the same token count (workload.py:145-153)
        per = span // len(ids)
        if per * len(ids) != span:
            raise ValueError("measured executor expects uniform doc token counts")
        return (per,) * len(ids)


@dataclass
class CalibratedExecutor:
    """Executor for ``sim.run`` whose costs are B200 *measurements* taken on one
    GPU (scripts/calibrate_costs.py): prefill time by cached-prefix level,
    host-tier and disk load time per byte, generation time by prefix length.
    Lets the reference policy project multi-instance runs (C4: 8 instances)
    that one GPU cannot host; results are modeled, and labeled as such."""

    costs: dict
    # per-byte cost of a memory-tier hit; None = the measured pinned-host-tier load.
    # C4 "P2P on" sets it to a peer-HBM fetch (K3p over NVLink) — the memory tier
    # then stands for the instances' pooled HBM
    memory_tier_s_per_byte: float | None = None

    def bind(self, config: SimConfig, cache: TierMirror) -> None:
        self.cfg = config
        c = self.costs
        if config.k != c["k"]:
            raise ValueError(f"costs were measured for k={c['k']}, config has k={config.k}")

    def serve(self, d: Dispatch) -> tuple[float, float]:
        c = self.costs
        prefill = c["prefill_s_by_cached_docs"][d.best]
        if d.best == 0:
            return 0.0, prefill
        mem = c["host_tier_load_s_per_byte"] if self.memory_tier_s_per_byte is None else self.memory_tier_s_per_byte
        per = mem if d.tier is Tier.MEMORY else c["disk_read_verify_s_per_byte"]
        return per * d.size_bytes, prefill

    def generation_time(self, task: GenTask) -> float:
        return self.costs["generation_s_by_docs"][len(task.prefix) - 1]

    def generated(self, task: GenTask) -> None:
        pass


def summarize(records, access_log=None) -> dict:
    """TTFT percentiles (both definitions) and throughput of a run."""
    lat = np.array([r.first_token - r.arrival for r in records])
    ttft = np.array([r.kv_load + r.prefill + r.network_delay for r in records])
    # throughput over the SUM of per-try makespans (reference build_report, sim.py:226-240):
    # the tries run back to back on the same clock origin, so one span would double-count
    tries: dict[int, list] = {}
    for r in records:
        tries.setdefault(getattr(r, "try_index", 1), []).append(r)
    span = sum(max(r.first_token for r in g) - min(r.arrival for r in g) for g in tries.values())
    origins: dict[str, int] = {}
    for r in records:
        for o in r.origins:
            origins[o] = origins.get(o, 0) + 1
    out = {
        "queries": len(records),
        "qps": len(records) / span if span > 0 else 0.0,
        "latency_ms": {"p50": float(np.percentile(lat, 50) * 1e3), "p99": float(np.percentile(lat, 99) * 1e3)},
        "ttft_ms": {"p50": float(np.percentile(ttft, 50) * 1e3), "p99": float(np.percentile(ttft, 99) * 1e3)},
        "origins": dict(sorted(origins.items())),
    }
    if access_log:
        out["store_outcomes"] = {}
        for a in access_log:
            out["store_outcomes"][a.outcome] = out["store_outcomes"].get(a.outcome, 0) + 1
    return out
