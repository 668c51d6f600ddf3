"""C5 at full depth on ONE B200 (SURVEY §8d config 5 without the tensor split).

Llama-3-70B shape, all 80 layers, random-init bf16 weights (141 GB: a whole
70B instance fits one B200's HBM), 20 documents x 1024 tokens + a 64-token query:

* document-KV generation of the 20-doc composite (20480 tokens, 6.7 GB of KV),
  written in the blob layout, FNV-hashed on the GPU, copied to the pinned host tier;
* first-token TTFT of the same query three ways on the same GPU:
  full-prompt prefill (20544 tokens, the no-cache baseline), cached prefix from the
  pinned host tier (6.7 GB layer-streamed H2D + K3 unpack overlapped with the
  query's layers), cached prefix resident in the HBM tier (loads nothing);
* K3 unpack bandwidth sweep over the cached-token count (1..20 documents).

The reference's TTFT law is kv_load + prefill (costs.py:125-144); its load is
bytes / tier bandwidth (costs.py:102-108).  Timed with CUDA events on the
launching stream (device) and wall clock around the public prefill_batch call
(host view, first token read back).

    python scripts/c5_full.py > profiles/r2_c5_full_depth.json
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

from paper_2504_11765_b200.engine import Engine, kv_unpack, pack_unpack_jobs
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import KvKey, LookupResult, Outcome
from paper_2504_11765_b200.model import combo_tokens

K, DOC, Q = 20, 1024, 64
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 80
spec = get_spec("llama-3-70b", layers)
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
free0, total = torch.cuda.mem_get_info()
n_ctx = K * DOC + Q
kvb = spec.kv_bytes_per_token()
comp_bytes = kvb * K * DOC
wbytes = 2 * (spec.nonembedding_params() + 2 * spec.vocab * spec.hidden)
need = wbytes + 2 * comp_bytes + kvb * (n_ctx + 256) + 6 * 2**30
if need > free0:
    print(json.dumps({"error": f"needs ~{need / 1e9:.1f} GB, {free0 / 1e9:.1f} GB free"}))
    sys.exit(0)
t0 = time.perf_counter()
eng = Engine(spec, seed=0, pool_tokens=n_ctx + 256, device_cache_bytes=comp_bytes + kvb * 64)
torch.cuda.synchronize()
init_s = time.perf_counter() - t0
gen = KvGenerator(eng, keep_on_device=True)
ids = tuple(range(101, 101 + K))
key = KvKey(spec.profile().model_hash, ids)

# ---- document-KV generation of the composite (one row-deterministic prefill)
toks = gen.tokens(ids, [DOC] * K)
for _ in range(1):  # warm-up (workspace growth, tensor maps)
    out = eng.generate_doc_kv(toks)
    del out
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
kv = eng.generate_doc_kv(toks)
e1.record()
torch.cuda.synchronize()
gen_ms = e0.elapsed_time(e1)
gen_flops = spec.prefill_flops(len(toks), 0, with_head=False)
del kv
torch.cuda.empty_cache()
t0 = time.perf_counter()
blob = gen.generate(ids, [DOC] * K)  # prefill + GPU FNV + D2H to pinned host + HBM-tier insert
torch.cuda.synchronize()
gen_wall = time.perf_counter() - t0
torch.cuda.empty_cache()

qt = query_tokens(7, Q, spec.vocab)


def ttft(req, reps):
    ts, dev = [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        a.record()
        r = prefill_batch(eng, [req], timed=False, use_graph=False)
        b.record()
        first = int(r.next_token[0])
        ts.append(time.perf_counter() - t)
        torch.cuda.synchronize()
        dev.append(a.elapsed_time(b))
    return {"wall_ms_p50": float(np.median(ts) * 1e3), "wall_ms_min": float(min(ts) * 1e3),
            "device_ms_p50": float(np.median(dev)), "n": reps, "first_token": first}


res = {}
hbm = PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blob, 0), None, qt, key)
host = PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blob, 0), None, qt, None)
full = PrefillRequest(LookupResult(Outcome.MISS), combo_tokens(ids, [DOC] * K, spec.vocab), qt)
for name, req, reps in (("warm_hbm", hbm, 10), ("warm_host", host, 6), ("full_prefill", full, 3)):
    ttft(req, 1)
    res[name] = ttft(req, reps)
    torch.cuda.empty_cache()
same = len({res[k]["first_token"] for k in res}) == 1

# ---- greedy decode after the first token (decode.py): the HBM-tier query, 32 steps
from paper_2504_11765_b200 import decode as _decode

dec = None
try:
    seqs = _decode.start(eng, [hbm], 40)
    _decode.step(eng, seqs)
    prev = torch.tensor([s.last for s in seqs], dtype=torch.int32, device=eng.device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(32):
        prev = _decode.step(eng, seqs, sync=False, dev_tokens=prev).clone()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 32
    step_bytes = 2 * (spec.nonembedding_params() + spec.vocab * spec.hidden) + kvb * (n_ctx + 17)
    dec = {"batch": 1, "ms_per_token": ms, "tokens_per_s": 1e3 / ms, "bytes_per_step": step_bytes,
           "frac_of_hbm": step_bytes / ms / 1e6 / peaks["hbm_gbs"]}
    for s_ in seqs:
        _decode.retire(eng, s_)
except Exception as exc:  # the measurements above stand on their own
    dec = {"error": f"{type(exc).__name__}: {exc}"[:300]}
torch.cuda.empty_cache()

# ---- K3 sweep: cached tokens 1..20 documents, staged payload -> pool (HBM-bound)
rows = []
dev_payload = eng.stage(blob.payload_tensor())
torch.cuda.synchronize()
for nd in (1, 2, 5, 10, 20):
    n = nd * DOC
    numel = spec.layers * 2 * spec.kv_heads * n * spec.head_dim
    src = dev_payload[:numel]
    blocks = eng.pool.alloc_blocks(eng.pool.blocks_for(n))
    bt = torch.tensor(blocks, dtype=torch.int32, device=eng.device)
    jobs = [(src, n, 0)]
    jd = pack_unpack_jobs(jobs).to(eng.device)
    for _ in range(3):
        kv_unpack(eng.pool, jobs, bt, jobs_dev=jd)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        kv_unpack(eng.pool, jobs, bt, jobs_dev=jd)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    nbytes = 2 * numel * 2
    rows.append({"docs": nd, "tokens": n, "payload_GB": numel * 2 / 1e9, "unpack_ms": ms,
                 "unpack_gbps": nbytes / ms / 1e6, "frac_of_hbm": nbytes / ms / 1e6 / peaks["hbm_gbs"]})
    eng.pool.release(blocks)

print(json.dumps({
    "config": f"C5 llama-3-70b-shaped, {layers} layers, TP=1 (whole instance on one B200), random-init bf16, "
              f"{K} docs x {DOC} tok + {Q}-tok query",
    "weights_GB": wbytes / 1e9, "init_s": init_s, "composite_kv_GB": comp_bytes / 1e9,
    "generation": {"tokens": len(toks), "device_ms": gen_ms, "tflops": gen_flops / gen_ms / 1e9,
                   "frac_of_burst": gen_flops / gen_ms / 1e9 / peaks["bf16_tflops"],
                   "wall_ms_with_fnv_d2h": gen_wall * 1e3},
    "ttft_ms": res, "same_first_token": same, "decode": dec,
    "speedup_vs_full_prefill": {k: res["full_prefill"]["wall_ms_p50"] / res[k]["wall_ms_p50"]
                                for k in ("warm_hbm", "warm_host")},
    "k3_sweep": rows, "hbm_peak_gbs": peaks["hbm_gbs"],
}))
