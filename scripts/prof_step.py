"""Run a few bench steps (HBM-resident cached KV; C3 by default) between
cudaProfilerStart/Stop for `ncu --profile-from-start off` captures."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import argparse
import numpy as np
import torch
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import KvKey, LookupResult, Outcome
from paper_2504_11765_b200.workload import zipf_stream

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama-3-8b")
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--graph", type=int, default=1, help="1: CUDA-graph replay (the bench step), 0: eager")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--full", action="store_true", help="full-prompt prefill instead of cached")
a = ap.parse_args()
spec = get_spec(a.model)
B = a.batch
n_ctx = a.k * 512
eng = Engine(spec, seed=0, pool_tokens=B * (n_ctx + 128) + 4096, device_cache_bytes=(B + 2) * spec.kv_bytes_per_token() * n_ctx)
gen = KvGenerator(eng)
items = zipf_stream(10000, 1.0, B, seed=1, k=a.k, q_tokens=64, doc_tokens=512)
reqs = []
for it in items:
    blob = gen.generate(it.doc_ids, it.doc_tokens)
    key = KvKey(spec.profile().model_hash, it.doc_ids)
    q = query_tokens(it.query_id, 64, spec.vocab)
    if a.full:
        reqs.append(PrefillRequest(LookupResult(Outcome.MISS), gen.tokens(it.doc_ids, it.doc_tokens), q))
    else:
        reqs.append(PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blob, 0), None, q, key))
for _ in range(2):
    prefill_batch(eng, reqs, timed=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.steps):
    prefill_batch(eng, reqs, timed=False, use_graph=bool(a.graph))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
