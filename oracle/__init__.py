"""CPU oracle for the Shared RAG-DCache hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product (`paper_2504_11765_b200`) imports this package.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs use it, and only as the checker or the timed CPU
baseline, never as a fallback for the CUDA path.

Contents
  codec_ref.c / codec_ref.py  byte/integer restatement of ragdcache.codec
                              (FNV-1a, splitmix keystream, header layout) in C
                              and numpy; pinned against the reference's golden
                              vectors in tests/golden/ (tests/test_oracle.py).
  store_ref.py                restatement of the KvStore outcome/LRU law
                              (store.py:159-309) as a pure-Python state machine.
  llama_ref.py                fp32 PyTorch-CPU restatement of the document
                              prefill and prefill-with-cached-prefix numerics.
                              The reference has NO numerics for this path (its
                              payloads are noise, codec.py:3-6; prefill is the
                              cost model costs.py:82-99), so KV/logit parity is
                              "parity unpinned" by the reference: it is pinned
                              only by this restatement plus the reference's
                              prefix semantics (prefetch.py:6-8, costs.py:3-7,
                              89-99, sim.py:414-431) and the self-consistency
                              checks in tests/ (cached == full prefill).
"""
