"""Dev: per-kernel-class device time of a single-query prefill (eager, profiled)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import KvKey, LookupResult, Outcome
from paper_2504_11765_b200.workload import zipf_stream
spec = get_spec(sys.argv[1] if len(sys.argv) > 1 else "llama-3.2-1b")
eng = Engine(spec, seed=0, pool_tokens=8192, device_cache_bytes=1 << 30)
gen = KvGenerator(eng)
it = zipf_stream(10000, 1.0, 1, seed=1, k=5, q_tokens=64, doc_tokens=512)[0]
blob = gen.generate(it.doc_ids, it.doc_tokens)
key = KvKey(spec.profile().model_hash, it.doc_ids)
req = PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blob, 0), None, query_tokens(0, 64, spec.vocab), key)
for _ in range(5): prefill_batch(eng, [req], timed=False, use_graph=False)
torch.cuda.synchronize()
eng.model.collect(); eng.model.profile(True)
ev = []
for _ in range(10): prefill_batch(eng, [req], timed=False, use_graph=False, unpack_events=ev)
torch.cuda.synchronize()
eng.model.profile(False)
c = eng.model.collect()
print({k: round(v["ms"] / 10, 4) for k, v in c.items()}, "unpack", sum(a.elapsed_time(b) for a, b in ev) / 10)
for g in (False, True):
    ts = []
    for _ in range(20):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = prefill_batch(eng, [req], timed=False, use_graph=g); int(r.next_token[0])
        ts.append(time.perf_counter() - t0)
    print("graph" if g else "eager", "ttft ms p50", np.percentile(ts, 50) * 1e3)
# device-only timing of the graph replay
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): prefill_batch(eng, [req], timed=False, use_graph=True)
e1.record(); torch.cuda.synchronize()
print("graph device+host pipelined ms/query", e0.elapsed_time(e1) / 20)
# one profiled forward for ncu (--profile-from-start off)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
prefill_batch(eng, [req], timed=False, use_graph=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
