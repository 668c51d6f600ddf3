"""Query workloads: Zipf document locality and arrival processes.

Same streams as ``ragdcache.workload`` (reference workload.py:112-154,
:253-270) for the same seeds — the draws go through numpy's PCG64 in the same
order, so a workload built here is the workload the reference simulator sees.
Locality analysis and traces (workload.py:50-98, 157-250) are out of scope
(figure reproduction only).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

DEFAULT_Q_TOKENS = 16
DEFAULT_DOC_TOKENS = 120


@dataclass(frozen=True)
class WorkItem:
    """One query with pre-resolved documents (workload.py:28-47)."""

    query_id: int
    q_tokens: int
    doc_ids: tuple[int, ...] | None = None
    doc_tokens: tuple[int, ...] | None = None
    embedding: np.ndarray | None = None

    def __post_init__(self) -> None:
        if (self.doc_ids is None) == (self.embedding is None):
            raise ValueError("exactly one of doc_ids / embedding must be present")
        if self.q_tokens < 1:
            raise ValueError("q_tokens must be >= 1")
        if self.doc_ids is not None:
            if not self.doc_ids:
                raise ValueError("doc_ids must be non-empty when present")
            if self.doc_tokens is None or len(self.doc_tokens) != len(self.doc_ids):
                raise ValueError("doc_tokens must match doc_ids length")


def zipf_probabilities(n_docs: int, s: float) -> np.ndarray:
    if n_docs < 1:
        raise ValueError("n_docs must be >= 1")
    if s < 0:
        raise ValueError("s must be >= 0")
    w = np.arange(1, n_docs + 1, dtype=np.float64) ** (-s)
    return w / w.sum()


def zipf_stream(n_docs: int, s: float, n_queries: int, seed: int, k: int = 1,
                q_tokens: int = DEFAULT_Q_TOKENS, doc_tokens: int = DEFAULT_DOC_TOKENS) -> list[WorkItem]:
    """Each query retrieves k distinct docs drawn i.i.d. Zipf(s) over ids 1..n_docs;
    a duplicate within a row is redrawn in place, left to right."""
    if not 1 <= k <= n_docs:
        raise ValueError("k must be in 1..n_docs")
    cdf = np.cumsum(zipf_probabilities(n_docs, s))
    cdf[-1] = 1.0
    rng = np.random.default_rng(seed)

    def sample(m: int) -> np.ndarray:
        return np.searchsorted(cdf, rng.random(m), side="right") + 1

    picks = np.stack([sample(n_queries) for _ in range(k)], axis=1)
    if k > 1:
        for r in range(n_queries):
            used: set[int] = set()
            for c in range(k):
                while int(picks[r, c]) in used:
                    picks[r, c] = sample(1)[0]
                used.add(int(picks[r, c]))
    toks = (doc_tokens,) * k
    return [WorkItem(query_id=i, q_tokens=q_tokens, doc_ids=tuple(int(x) for x in picks[i]), doc_tokens=toks)
            for i in range(n_queries)]


def poissonize(items: Sequence[WorkItem], rate: float, seed: int) -> list[tuple[float, WorkItem]]:
    """Exponential inter-arrival gaps of mean 1/rate (workload.py:253-262)."""
    if rate <= 0:
        raise ValueError("rate must be positive")
    gaps = np.random.default_rng(seed).exponential(scale=1.0 / rate, size=len(items))
    return [(float(t), it) for t, it in zip(np.cumsum(gaps), items)]


def uniform_arrivals(items: Sequence[WorkItem], rate: float) -> list[tuple[float, WorkItem]]:
    if rate <= 0:
        raise ValueError("rate must be positive")
    dt = 1.0 / rate
    return [(dt * (i + 1), it) for i, it in enumerate(items)]


class TraceError(ValueError):
    """A malformed work trace (workload.py:190-231)."""


def save_trace(items: Iterable[WorkItem], path: str | Path) -> None:
    """One JSON object per line, keys sorted (workload.py:234-250)."""
    lines = []
    for it in items:
        if it.doc_ids is None:
            raise ValueError("only doc-id items can be saved to a trace")
        lines.append(json.dumps({"query_id": it.query_id, "doc_ids": list(it.doc_ids), "q_tokens": it.q_tokens,
                                 "doc_tokens": list(it.doc_tokens)}, sort_keys=True))
    Path(path).write_text("".join(line + "\n" for line in lines), encoding="utf-8")


def load_trace(path: str | Path) -> list[WorkItem]:
    """Inverse of save_trace; missing token counts take the module defaults and
    a missing query_id the 0-based line number (workload.py:190-231)."""
    items = []
    for lineno, line in enumerate(Path(path).read_text(encoding="utf-8").splitlines(), start=1):
        if not line.strip():
            continue
        try:
            obj = json.loads(line)
        except json.JSONDecodeError as exc:
            raise TraceError(f"{path}:{lineno}: invalid JSON: {exc}") from exc
        try:
            doc_ids = tuple(int(d) for d in obj["doc_ids"])
        except (KeyError, TypeError, ValueError) as exc:
            raise TraceError(f"{path}:{lineno}: field 'doc_ids': {exc}") from exc
        raw = obj.get("doc_tokens")
        doc_tokens = (DEFAULT_DOC_TOKENS,) * len(doc_ids) if raw is None else tuple(int(t) for t in raw)
        if len(doc_tokens) != len(doc_ids):
            raise TraceError(f"{path}:{lineno}: field 'doc_tokens': length {len(doc_tokens)} does not match "
                             f"{len(doc_ids)} doc_ids")
        try:
            items.append(WorkItem(query_id=int(obj.get("query_id", lineno - 1)),
                                  q_tokens=int(obj.get("q_tokens", DEFAULT_Q_TOKENS)), doc_ids=doc_ids,
                                  doc_tokens=doc_tokens))
        except ValueError as exc:
            raise TraceError(f"{path}:{lineno}: {exc}") from exc
    if not items:
        raise TraceError(f"{path}: no work items")
    return items
