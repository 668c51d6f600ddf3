"""Full-depth parity at the bench shapes (C2 16 layers, C3 32 layers, full width)
against the fp32 oracle, plus the bench step itself (every query of one
CUDA-graph-replayed HBM-tier batch) and the first-token agreement statistics
SURVEY H-h asks for.

Tolerance (north_star): rel err = max|gpu - oracle| / max|oracle| <= 2e-2 on
document KV and logits.  First token: the device argmax must equal the
oracle's argmax, except where the oracle's own top-2 are closer than the
measured logit error (a near-tie) — there the device pick must be one of the
oracle's near-tied tokens.  The agreement rate and the margin distribution are
written to gpurun_out/parity_argmax.json (committed copies under profiles/).
"""

import json
import os
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.llama_ref import OracleModel, rel_err
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import KvKey, KvStore, Outcome
from paper_2504_11765_b200.workload import zipf_stream

pytestmark = pytest.mark.gpu

TOL = 2e-2
OUT = Path(os.environ.get("GRAFT_REPO_ROOT", Path(__file__).resolve().parents[1])) / "gpurun_out"
CONFIGS = {"C2": ("llama-3.2-1b", 5, 32), "C3": ("llama-3-8b", 10, 16)}  # model, docs per query, bench batch
_REPORT: dict = {}


def _record(name, entry):
    _REPORT[name] = entry
    OUT.mkdir(exist_ok=True)
    (OUT / "parity_argmax.json").write_text(json.dumps(_REPORT, indent=1))


def first_token_verdict(gpu_logits: torch.Tensor, gpu_arg: int, ref: torch.Tensor) -> dict:
    """Compare one query's first token with the oracle's; returns the record
    (raises on a disagreement that is not a near-tie)."""
    g = gpu_logits.float().cpu()
    abs_err = float((g - ref).abs().max())
    top = torch.topk(ref, 2)
    margin = float(top.values[0] - top.values[1])
    agree = gpu_arg == int(top.indices[0])
    rec = {"agree": agree, "margin": margin, "abs_err": abs_err, "rel_err": rel_err(g, ref)}
    if not agree:
        # allowed only when the oracle itself cannot separate the two within the error
        gap = float(ref.max() - ref[gpu_arg])
        assert gap <= 2 * abs_err, f"first token {gpu_arg} vs oracle {int(top.indices[0])}: gap {gap:.4f} " \
                                   f"> 2x logit error {abs_err:.4f} (margin {margin:.4f})"
    return rec


@pytest.fixture(scope="module", params=["C2", "C3"])
def bench_setup(request, tmp_path_factory):
    """One engine per config with the bench's warm batch: composites generated on
    the GPU, put in a KvStore (memory tier), resident in the HBM tier."""
    name = request.param
    model, k, B = CONFIGS[name]
    spec = get_spec(model)
    comp = spec.kv_bytes_per_token() * k * 512
    eng = Engine(spec, seed=0, pool_tokens=B * (k * 512 + 128) + 4096, device_cache_bytes=(B + 2) * comp)
    gen = KvGenerator(eng, keep_on_device=True)
    items = zipf_stream(10_000, 1.0, B, seed=1, k=k, q_tokens=64, doc_tokens=512)
    prof = spec.profile()
    keys = [KvKey(prof.model_hash, it.doc_ids) for it in items]
    store = KvStore(tmp_path_factory.mktemp(f"store_{name}"), memory_capacity_bytes=(B + 1) * (comp + 4096))
    for it, key in zip(items, keys):
        store.put(key, gen.generate(it.doc_ids, it.doc_tokens))
    torch.cuda.synchronize()
    orc = OracleModel(eng.weights, n_threads=os.cpu_count())
    yield name, spec, eng, gen, items, keys, store, orc
    del orc, eng
    torch.cuda.empty_cache()


def test_full_depth_composite_kv_and_logits(bench_setup):
    """One composite of the bench (k x 512 tokens, every layer) + its 64-token
    query: device KV vs oracle KV, device logits (query prefilled over the
    device-generated cached KV) vs the oracle's full-prompt logits."""
    name, spec, eng, gen, items, keys, store, orc = bench_setup
    it, key = items[0], keys[0]
    look = store.get(key)
    assert look.outcome is Outcome.MEMORY_HIT
    n = look.blob.header.token_count
    q = query_tokens(it.query_id, 64, spec.vocab)
    r = prefill_batch(eng, [PrefillRequest(look, None, q, None)], timed=False)   # host tier -> H2D -> K3 -> prefill
    torch.cuda.synchronize()
    kv_ref, lg_ref = orc.forward(np.concatenate([gen.tokens(it.doc_ids, it.doc_tokens), q]))
    kv_dev = look.blob.payload_tensor().view(torch.bfloat16).view(spec.layers, 2, spec.kv_heads, n, spec.head_dim)
    e_kv = rel_err(kv_dev, kv_ref[:, :, :, :n])
    e_lg = rel_err(r.logits[0], lg_ref)
    rec = first_token_verdict(r.logits[0], int(r.next_token[0]), lg_ref)
    _record(f"{name}_full_depth", {"layers": spec.layers, "cached_tokens": n, "kv_rel_err": e_kv,
                                   "logits_rel_err": e_lg, **rec})
    assert e_kv <= TOL, f"{name} KV rel err {e_kv:.3e}"
    assert e_lg <= TOL, f"{name} logits rel err {e_lg:.3e}"


def test_bench_step_every_query_matches_oracle(bench_setup):
    """The bench's value step exactly: B KvStore.get MEMORY_HITs, HBM-tier KV,
    one CUDA-graph replay; every query's logits and first token against the
    oracle prefilling the same 64 tokens over the same cached KV."""
    name, spec, eng, gen, items, keys, store, orc = bench_setup
    B = len(items)
    reqs = [PrefillRequest(store.get(k), None, query_tokens(it.query_id, 64, spec.vocab), k)
            for it, k in zip(items, keys)]
    prefill_batch(eng, reqs, timed=False)                 # capture
    reqs = [PrefillRequest(store.get(k), None, query_tokens(it.query_id, 64, spec.vocab), k)
            for it, k in zip(items, keys)]
    r = prefill_batch(eng, reqs, timed=False)              # replay (the timed path)
    logits, nxt = r.logits.clone(), r.next_token.clone()
    torch.cuda.synchronize()
    recs = []
    for i, (it, req) in enumerate(zip(items, reqs)):
        n = req.lookup.blob.header.token_count
        past = req.lookup.blob.payload_tensor().view(torch.bfloat16).view(
            spec.layers, 2, spec.kv_heads, n, spec.head_dim)
        _, ref = orc.forward(req.new_tokens, past, n)
        rec = first_token_verdict(logits[i], int(nxt[i]), ref)
        assert rec["rel_err"] <= TOL, f"{name} query {i}: logits rel err {rec['rel_err']:.3e}"
        recs.append(rec)
    agree = sum(r_["agree"] for r_ in recs) / B
    margins = sorted(r_["margin"] for r_ in recs)
    _record(f"{name}_bench_step", {"queries": B, "agreement": agree, "max_rel_err": max(r_["rel_err"] for r_ in recs),
                                   "max_abs_err": max(r_["abs_err"] for r_ in recs), "margins": margins})
    assert agree >= 0.9, f"{name}: first-token agreement {agree:.2f}"


def test_first_token_agreement_64_queries(bench_setup):
    """>= 64 queries over the bench composites (4 query streams each): the
    agreement rate and margin histogram of SURVEY H-h."""
    name, spec, eng, gen, items, keys, store, orc = bench_setup
    if name != "C2":
        pytest.skip("64-query statistics at C2 (the C3 oracle costs ~1 TFLOP per query)")
    recs = []
    for rep in range(2):
        reqs = [PrefillRequest(store.get(k), None, query_tokens(5000 + 100 * rep + i, 64, spec.vocab), k)
                for i, k in enumerate(keys)]
        r = prefill_batch(eng, reqs, timed=False, use_graph=False)
        logits, nxt = r.logits.clone(), r.next_token.clone()
        torch.cuda.synchronize()
        for i, req in enumerate(reqs):
            n = req.lookup.blob.header.token_count
            past = req.lookup.blob.payload_tensor().view(torch.bfloat16).view(
                spec.layers, 2, spec.kv_heads, n, spec.head_dim)
            _, ref = orc.forward(req.new_tokens, past, n)
            recs.append(first_token_verdict(logits[i], int(nxt[i]), ref))
    assert len(recs) >= 64
    agree = sum(r_["agree"] for r_ in recs) / len(recs)
    m = np.array([r_["margin"] for r_ in recs])
    e = np.array([r_["abs_err"] for r_ in recs])
    hist, edges = np.histogram(m / np.maximum(e, 1e-9), bins=[0, 1, 2, 4, 8, 16, 32, 1e9])
    _record(f"{name}_agreement_{len(recs)}", {"queries": len(recs), "agreement": agree,
                                              "margin_over_err_hist": dict(zip([f"<{x:g}" for x in edges[1:]],
                                                                               hist.tolist())),
                                              "median_margin": float(np.median(m)), "median_abs_err": float(np.median(e))})
    assert agree >= 0.9
