"""Decode step time of the C3 bench batch (16 sequences over ~5.2k cached tokens) for A/B of
library variants (RDKV_LIB=...): ms per step over 24 steps, the per-class attention time
(eager profile), and a digest of the generated tokens (variants must agree)."""
import hashlib
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_11765_b200 import decode
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest
from paper_2504_11765_b200.store import KvKey, LookupResult, Outcome
from paper_2504_11765_b200.workload import zipf_stream

spec = get_spec(sys.argv[1] if len(sys.argv) > 1 else "llama-3-8b")
B, n_ctx = 16, 10 * 512
eng = Engine(spec, seed=0, pool_tokens=B * (n_ctx + 192) + 4096, device_cache_bytes=(B + 2) * spec.kv_bytes_per_token() * n_ctx)
gen = KvGenerator(eng)
reqs = []
for it in zipf_stream(10000, 1.0, B, seed=1, k=10, q_tokens=64, doc_tokens=512):
    blob = gen.generate(it.doc_ids, it.doc_tokens)
    key = KvKey(spec.profile().model_hash, it.doc_ids)
    eng.make_resident(key, blob.device if blob.device is not None else eng.stage(blob.payload_tensor()), n_ctx)
    reqs.append(PrefillRequest(LookupResult(Outcome.MEMORY_HIT, None, 0), None, query_tokens(it.query_id, 64, spec.vocab), key))
torch.cuda.synchronize()
out = {}
for rep in range(2):
    seqs = decode.start(eng, reqs, 64)
    for _ in range(4):
        decode.step(eng, seqs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(24):
        decode.step(eng, seqs, sync=False)
    e1.record()
    torch.cuda.synchronize()
    out[f"ms_per_step_{rep}"] = round(e0.elapsed_time(e1) / 24, 4)
    eng.model.collect()
    eng.model.profile(True)
    for _ in range(8):
        decode.step(eng, seqs, sync=False)
    torch.cuda.synchronize()
    eng.model.profile(False)
    cl = eng.model.collect()
    out[f"attention_ms_{rep}"] = round(cl["attention"]["ms"] / 8, 4)
    decode.step(eng, seqs)
    for s in seqs:
        decode.retire(eng, s)
first = decode.generate(eng, reqs[:4], 12)
out["tokens_digest"] = hashlib.sha1(json.dumps(first).encode()).hexdigest()[:12]
print(json.dumps(out))
