"""Measure the per-query B200 costs the reference scheduling policy needs
(sim.Executor: serve = kv_load + prefill, generation_time), for one model and
k docs x N tokens + q-token queries.  Output feeds serving.CalibratedExecutor,
which lets sim.run project multi-instance (C4) behaviour from one GPU.

    python scripts/calibrate_costs.py --model llama-3-8b --k 10 > profiles/r1_b200_costs_8b.json
"""
import argparse
import json
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2504_11765_b200 import _lib
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import combo_tokens, get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import GpuVerifier, KvKey, KvStore, LookupResult, Outcome


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-3-8b")
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--doc-tokens", type=int, default=512)
    ap.add_argument("--q-tokens", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    spec = get_spec(a.model)
    k, N, q = a.k, a.doc_tokens, a.q_tokens
    comp = spec.kv_bytes_per_token() * k * N
    eng = Engine(spec, seed=0, pool_tokens=2 * (k * N + q) + 4096, device_cache_bytes=2 * comp)
    gen = KvGenerator(eng, keep_on_device=True)
    docs = tuple(range(101, 101 + k))
    prof = spec.profile()
    qt = query_tokens(7, q, spec.vocab)

    def ttft(req):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = prefill_batch(eng, [req], timed=False)
        int(r.next_token[0])
        return time.perf_counter() - t0

    out = {"model": a.model, "k": k, "doc_tokens": N, "q_tokens": q, "composite_bytes": comp}
    # generation of every prefix level (span j*N) — GPU prefill, GPU FNV, D2H into the host tier
    gen_s, blobs = [], []
    for j in range(1, k + 1):
        gen.generate(docs[:j], (N,) * j)  # warm
        ts = []
        for _ in range(max(1, a.reps // 2)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            b = gen.generate(docs[:j], (N,) * j)
            ts.append(time.perf_counter() - t0)
        gen_s.append(float(np.median(ts)))
        blobs.append(b)
    out["generation_s_by_docs"] = gen_s
    # prefill over an HBM-resident prefix of j docs: new tokens = remaining docs + query (sim.py:420-422)
    pre_s = []
    for j in range(0, k + 1):
        rest = combo_tokens(docs[j:], (N,) * (k - j), spec.vocab)
        new = np.concatenate([rest, qt]) if len(rest) else qt
        if j == 0:
            req = PrefillRequest(LookupResult(Outcome.MISS), np.zeros(0, np.int32), new)
        else:
            req = PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blobs[j - 1], 0), None, new,
                                 KvKey(prof.model_hash, docs[:j]))
        ttft(req)
        pre_s.append(float(np.median([ttft(req) for _ in range(a.reps)])))
    out["prefill_s_by_cached_docs"] = pre_s
    # host-tier load of the full composite (layer-streamed H2D + unpack), as extra time over the HBM-resident case
    host = PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blobs[-1], 0), None, qt, None)
    ttft(host)
    out["host_tier_load_s_per_byte"] = max(0.0, float(np.median([ttft(host) for _ in range(a.reps)])) - pre_s[k]) / comp
    # cold disk: aligned parallel read + GPU FNV verify (page cache dropped)
    root = Path(tempfile.mkdtemp(prefix="rdkv_cal_"))
    store = KvStore(root, 0, verifier=GpuVerifier(eng.device))
    key = KvKey(prof.model_hash, docs)
    store.put(key, blobs[-1])
    ts = []
    for _ in range(3):
        _lib.lib().rdkv_drop_page_cache(str(store.path_of(key)).encode())
        t0 = time.perf_counter()
        look = store.get(key)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        assert look.outcome is Outcome.DISK_HIT
    out["disk_read_verify_s_per_byte"] = float(np.median(ts)) / comp
    print(json.dumps(out))


if __name__ == "__main__":
    main()
