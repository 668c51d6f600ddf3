"""Dev: C3 (Llama-3-8B-shaped) end-to-end on one GPU: doc-KV generation of a
10x512 composite, cached-prefix query prefill vs full prefill, a 2-layer
oracle cross-check, and step throughput at batch 16."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2504_11765_b200.engine import Engine, QueryRequest
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens, combo_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import KvKey, LookupResult, Outcome
from paper_2504_11765_b200.workload import zipf_stream

out = {}
# numerics at full width, truncated depth (oracle on CPU)
from oracle.llama_ref import OracleModel, rel_err, top1_margin
spec2 = get_spec("llama-3-8b", layers=2)
e2 = Engine(spec2, seed=0, pool_tokens=8192)
pre = combo_tokens([1, 2, 3], [512, 512, 512], spec2.vocab)
q = query_tokens(5, 64, spec2.vocab)
kv = e2.generate_doc_kv(pre)
lg, nx = e2.prefill([QueryRequest(q, kv, len(pre))])
torch.cuda.synchronize()
orc = OracleModel(e2.weights)
kref, ref = orc.forward(np.concatenate([pre, q]))
out["c3_2layer_logits_rel_err"] = rel_err(lg[0], ref)
out["c3_2layer_kv_rel_err"] = rel_err(kv.view(2, 2, 8, len(pre), 128).float().cpu(), kref[:, :, :, :len(pre)])
out["c3_2layer_argmax_match"] = int(nx[0]) == int(torch.argmax(ref))
out["c3_2layer_margin"] = top1_margin(ref)
del e2, orc
torch.cuda.empty_cache()

spec = get_spec("llama-3-8b")
B = 16
eng = Engine(spec, seed=0, pool_tokens=B * 5300 + 8192, device_cache_bytes=(B + 2) * spec.kv_bytes_per_token() * 5120)
gen = KvGenerator(eng)
items = zipf_stream(10000, 1.0, B, seed=1, k=10, q_tokens=64, doc_tokens=512)
torch.cuda.synchronize(); t0 = time.perf_counter()
blobs = [gen.generate(it.doc_ids, it.doc_tokens) for it in items]
torch.cuda.synchronize(); out["gen_s_per_composite"] = (time.perf_counter() - t0) / B
reqs = [PrefillRequest(LookupResult(Outcome.MEMORY_HIT, b, 0), None, query_tokens(it.query_id, 64, spec.vocab),
                       KvKey(spec.profile().model_hash, it.doc_ids)) for b, it in zip(blobs, items)]
for _ in range(2): prefill_batch(eng, reqs, timed=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): prefill_batch(eng, reqs, timed=False)
e1.record(); torch.cuda.synchronize()
out["c3_warm_qps_b16"] = B * 5 / (e0.elapsed_time(e1) / 1e3)
one = reqs[:1]
ts = []
for _ in range(10):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = prefill_batch(eng, one, timed=False); int(r.next_token[0]); ts.append(time.perf_counter() - t0)
out["c3_ttft_warm_ms_p50"] = float(np.median(ts) * 1e3)
full = [PrefillRequest(LookupResult(Outcome.MISS), gen.tokens(items[0].doc_ids, items[0].doc_tokens), query_tokens(0, 64, spec.vocab))]
ts = []
for _ in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = prefill_batch(eng, full, timed=False); int(r.next_token[0]); ts.append(time.perf_counter() - t0)
out["c3_ttft_full_ms_p50"] = float(np.median(ts) * 1e3)
print(json.dumps(out))
