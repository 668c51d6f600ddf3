"""C5 load-path sweep: K3 unpack bandwidth vs cached
tokens for one Llama-3-70B TP=4 rank (80 layers x 2 KV heads x dh 128: 80 KiB
per token), against the per-rank full-prefill time of the same tokens measured
on a layer-truncated 70B-shaped rank model and scaled to 80 layers.

    python scripts/k3_sweep.py > profiles/r1_k3_sweep_c5.json
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2504_11765_b200.engine import Engine, KvPool, QueryRequest, kv_unpack, pack_unpack_jobs
from paper_2504_11765_b200.model import combo_tokens, get_spec, init_weights, shard_weights, tp_spec

peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6650.0
full = get_spec("llama-3-70b")
rank = tp_spec(full, 4)                     # 2 KV heads, 16 q heads, ffn 7168 per rank
rows = []
pool = KvPool(rank, n_blocks=20480 // 64 + 8, block_size=64)
for n in (1024, 2048, 5120, 10240, 20480):
    numel = rank.layers * 2 * rank.kv_heads * n * rank.head_dim
    src = torch.randn(numel, device="cuda").bfloat16()
    blocks = pool.alloc(n)
    bt = torch.tensor(blocks, dtype=torch.int32, device="cuda")
    jd = pack_unpack_jobs([(src, n, 0)]).to("cuda")
    for _ in range(3):
        kv_unpack(pool, [(src, n, 0)], bt, jobs_dev=jd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        kv_unpack(pool, [(src, n, 0)], bt, jobs_dev=jd)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nbytes = 2 * numel * 2
    rows.append({"tokens": n, "payload_MiB": numel * 2 / 2**20, "unpack_ms": ms, "unpack_gbps": nbytes / ms / 1e6,
                 "frac_of_hbm_peak": nbytes / ms / 1e6 / peak})
    pool.release(blocks)
    del src
del pool
torch.cuda.empty_cache()
# full prefill of the same tokens on one TP rank, 4-layer truncation, scaled x20 to 80 layers
L = 4
spec4 = get_spec("llama-3-70b", L)
w = shard_weights(init_weights(spec4, 0), 0, 4)
eng = Engine(tp_spec(spec4, 4), weights=w, pool_tokens=20480 + 1024)
for r in rows:
    n = r["tokens"]
    toks = combo_tokens(list(range(1, n // 1024 + 1)), [1024] * (n // 1024), spec4.vocab)
    eng.generate_doc_kv(toks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.generate_doc_kv(toks)
    e1.record()
    torch.cuda.synchronize()
    r["rank_prefill_ms_80_layers_est"] = e0.elapsed_time(e1) * 80 / L
    r["prefill_over_load"] = r["rank_prefill_ms_80_layers_est"] / r["unpack_ms"]
print(json.dumps({"config": "C5 llama-3-70b TP=4, one rank (2 KV heads), K3 from HBM staging vs per-rank prefill "
                            "(no all-reduce; 4-layer truncation scaled to 80)", "hbm_peak_gbs": peak, "rows": rows}))
