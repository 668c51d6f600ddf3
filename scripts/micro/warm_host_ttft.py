"""Warm-host single-query TTFT: host time spent enqueueing the layer stream vs the total."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch
from paper_2504_11765_b200 import engine as E
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import LookupResult, Outcome

spec = get_spec("llama-3.2-1b")
eng = Engine(spec, seed=0, pool_tokens=16384, device_cache_bytes=0)
gen = KvGenerator(eng)
blob = gen.generate((1, 2, 3, 4, 5), (512,) * 5)
qt = query_tokens(1, 64, spec.vocab)
req = PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blob, 0), None, qt, None)
orig = E.LayerStreamer.launch
spent = []
def timed_launch(self, *a, **k):
    t0 = time.perf_counter(); r = orig(self, *a, **k); spent.append(time.perf_counter() - t0); return r
E.LayerStreamer.launch = timed_launch
ts = []
for i in range(30):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = prefill_batch(eng, [req], timed=False); int(r.next_token[0])
    ts.append(time.perf_counter() - t0)
print({"ttft_ms_p50": np.median(ts[5:]) * 1e3, "streamer_launch_ms_p50": np.median(spent[5:]) * 1e3})
