"""The KV generator plugin: ``generate() -> KvBlob`` backed by B200 prefill.

Replaces the reference's generator stand-in ``synth_blob`` (codec.py:188-224)
at its two call sites, ``prefetch.prepare`` (prefetch.py:150-152) and
``cli precompute`` (cli.py:161), under the plugin contract of
``SharedCacheService.get_or_generate`` (service.py:87-92): deterministic per
key, header matching the key, exceptions propagate to every waiter.

A call runs the document prefill over the ordered combination's concatenated
tokens (positions 0..n-1, prefetch.py:6-8) on the engine's GPU; the payload is
written by the QKV epilogue directly in the `.rdkv` layout, FNV-1a-hashed on
the GPU (codec.fnv1a64_device, bit-exact) while it is copied once into pinned
host memory (the memory tier's DMA-ready form), and wrapped without re-hashing.  The KV is also placed in the engine's HBM
tier (pool blocks) so a query dispatched to the same GPU loads nothing.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np
import torch

from .codec import KvBlob, fnv1a64_device, fnv1a64_device_async, make_header
from .engine import Engine
from .model import combo_tokens
from .store import KvKey


class KvGenerator:
    def __init__(self, engine: Engine, token_seed: int = 0, keep_on_device: bool = True) -> None:
        self.engine = engine
        self.profile = engine.spec.profile()
        self.token_seed = token_seed
        self.keep_on_device = keep_on_device
        self.copy_stream = engine.copy_stream  # D2H into the host tier (the runtime gives generation its own)

    def tokens(self, doc_ids: Sequence[int], doc_token_counts: Sequence[int]) -> np.ndarray:
        return combo_tokens(doc_ids, doc_token_counts, self.engine.spec.vocab, self.token_seed)

    def generate(self, doc_ids: Sequence[int], doc_token_counts: Sequence[int]) -> KvBlob:
        ids = tuple(int(d) for d in doc_ids)
        if not ids:
            raise ValueError("doc_ids must be non-empty")
        toks = self.tokens(ids, doc_token_counts)
        if len(toks) < 1:
            raise ValueError("token_count must be >= 1")
        eng = self.engine
        with torch.cuda.device(eng.device):
            # D2H into the host tier on the copy stream while the GPU hashes the payload
            return self._blob_from_device(ids, len(toks), eng.generate_doc_kv(toks))

    def _blob_from_device(self, ids: tuple[int, ...], n: int, kv: torch.Tensor) -> KvBlob:
        """Header + pinned host copy of a device payload, checksum on the GPU."""
        eng = self.engine
        raw = kv.view(torch.uint8)
        main = torch.cuda.current_stream(eng.device)
        cs = self.copy_stream
        cs.wait_stream(main)
        host = torch.empty(raw.numel(), dtype=torch.uint8, pin_memory=True)
        with torch.cuda.stream(cs):
            host.copy_(raw, non_blocking=True)
        raw.record_stream(cs)
        checksum = fnv1a64_device(raw)
        cs.synchronize()
        if self.keep_on_device:
            eng.make_resident(KvKey(self.profile.model_hash, ids), kv, n)
        return KvBlob.trusted(make_header(self.profile, ids, n, checksum), host)

    def generate_many(self, combos: Sequence[tuple[Sequence[int], Sequence[int]]],
                      hosts: Sequence[torch.Tensor] | None = None) -> list[KvBlob]:
        """``generate`` for several combinations as one pipeline: composite i's D2H into the
        host tier (copy engine) runs while composite i+1 is prefilled, and the checksums stay
        on the device until the end — no host synchronisation between composites.  Each blob
        is byte-identical to ``generate`` of the same combination.  ``hosts``: optional
        pinned uint8 buffers (one per combination, at least the payload size) to copy into."""
        eng = self.engine
        out = []
        with torch.cuda.device(eng.device):
            main = torch.cuda.current_stream(eng.device)
            cs = self.copy_stream
            # the checksum of composite i runs on a low-priority stream beside the prefill of
            # composite i+1 (it takes the SMs the prefill's kernels leave idle)
            if getattr(self, "_fnv_stream", None) is None:
                lo, _ = torch.cuda.Stream.priority_range()
                self._fnv_stream = torch.cuda.Stream(device=eng.device, priority=lo)
            fs = self._fnv_stream
            pending = []
            for ci, (doc_ids, counts) in enumerate(combos):
                ids = tuple(int(d) for d in doc_ids)
                toks = self.tokens(ids, counts)
                kv = eng.generate_doc_kv(toks)
                raw = kv.view(torch.uint8)
                fs.wait_stream(main)
                csum = fnv1a64_device_async(raw, stream=fs)
                raw.record_stream(fs)
                host = hosts[ci][: raw.numel()] if hosts is not None else \
                    torch.empty(raw.numel(), dtype=torch.uint8, pin_memory=True)
                cs.wait_stream(main)
                with torch.cuda.stream(cs):
                    host.copy_(raw, non_blocking=True)
                raw.record_stream(cs)
                if self.keep_on_device:
                    eng.make_resident(KvKey(self.profile.model_hash, ids), kv, len(toks))
                pending.append((ids, len(toks), csum, host))
            cs.synchronize()
            fs.synchronize()
            main.synchronize()
            for ids, n, csum, host in pending:
                out.append(KvBlob.trusted(make_header(self.profile, ids, n, int(csum.item()) & ((1 << 64) - 1)), host))
        return out

    def slice_prefix(self, full: torch.Tensor, n_full: int, n: int) -> torch.Tensor:
        """Payload of the first n tokens of a combination's payload [L][2][Hkv][n_full][dh]
        (one strided device copy)."""
        from . import _lib
        from .engine import _L

        s = self.engine.spec
        if n == n_full:
            return full
        out = torch.empty(s.layers * 2 * s.kv_heads * n * s.head_dim, dtype=torch.bfloat16, device=full.device)
        row = s.head_dim * 2
        _lib.check(_L().rdkv_memcpy_2d(out.data_ptr(), n * row, full.data_ptr(), n_full * row, n * row,
                                       s.layers * 2 * s.kv_heads,
                                       torch.cuda.current_stream(full.device).cuda_stream))
        return out

    def for_combination(self, doc_ids: Sequence[int], doc_token_counts: Sequence[int]):
        """Generator factory for every prefix of one ordered combination: the first
        ``generate()`` runs the combination's prefill once (row-deterministic), each
        prefix is then a slice of it — bit-identical to generating that prefix from
        scratch (prefetch.py:6-8), with one forward instead of k."""
        full_ids, full_counts = tuple(int(d) for d in doc_ids), tuple(int(c) for c in doc_token_counts)
        state: dict = {}

        def factory(prefix_ids, prefix_counts):
            ids, counts = tuple(int(d) for d in prefix_ids), tuple(int(c) for c in prefix_counts)
            if ids != full_ids[: len(ids)] or counts != full_counts[: len(ids)]:
                return self.for_prefix(ids, counts)  # not a prefix of this combination

            def generate() -> KvBlob:
                eng = self.engine
                with torch.cuda.device(eng.device):
                    if "kv" not in state:
                        state["kv"] = eng.generate_doc_kv(self.tokens(full_ids, full_counts))
                        state["n"] = sum(full_counts)
                    n = sum(counts)
                    return self._blob_from_device(ids, n, self.slice_prefix(state["kv"], state["n"], n))

            return generate

        return factory

    def for_prefix(self, doc_ids: Sequence[int], doc_token_counts: Sequence[int]) -> Callable[[], KvBlob]:
        """The ``generate`` callable for one key (prefetch.prepare / get_or_generate)."""
        ids, counts = tuple(doc_ids), tuple(doc_token_counts)
        return lambda: self.generate(ids, counts)

    __call__ = for_prefix
