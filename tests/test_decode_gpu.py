"""Decode phase (decode.py): greedy tokens after the first one, each
step one forward of one new token per live sequence over its pool-resident context.

Checked teacher-forced against the fp32 oracle (oracle/llama_ref.py) fed the GPU's own
tokens through its incremental path (past_kv): every step's logits within rel err 2e-2
and the argmax identical whenever the oracle's top-1 margin exceeds 4x the observed
logit error (the tolerance rule of test_prefill_gpu.py).  Continuous batching must give
every request the same checks whatever joins or leaves the batch, and return every pool
block and HBM-tier pin.
"""

import numpy as np
import pytest
import torch

from oracle.llama_ref import OracleModel, rel_err, top1_margin
from paper_2504_11765_b200 import decode
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import combo_tokens, get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest
from paper_2504_11765_b200.store import KvKey, LookupResult, Outcome

pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module", params=["tiny", "gqa-small-128"])
def setup(request):
    spec = get_spec(request.param)
    eng = Engine(spec, seed=2, pool_tokens=16384, block_size=64, device_cache_bytes=64 << 20)
    return spec, eng, OracleModel(eng.weights), KvGenerator(eng, keep_on_device=False)


def _request(spec, gen, eng, docs, ntok, qid, q_len, hbm: bool):
    """A cached-prefix query: the composite's KV from the generator, as a host-tier blob
    (unpacked into the pool) or resident in the HBM tier (pool blocks shared)."""
    blob = gen.generate(docs, ntok)
    key = KvKey(spec.profile().model_hash, tuple(docs))
    look = LookupResult(Outcome.MEMORY_HIT, blob, 0)
    if hbm:
        eng.make_resident(key, eng.stage(blob.payload_tensor()), int(sum(ntok)))
        torch.cuda.synchronize()
        look = LookupResult(Outcome.MEMORY_HIT, None, 0)
    prompt = np.concatenate([combo_tokens(docs, ntok, spec.vocab), query_tokens(qid, q_len, spec.vocab)])
    return PrefillRequest(look, None, query_tokens(qid, q_len, spec.vocab), key if hbm else None), prompt


class _Oracle:
    """Incremental fp32 decode fed the GPU's tokens (teacher forcing)."""

    def __init__(self, orc, prompt):
        self.orc = orc
        self.kv, self.logits = orc.forward(prompt)
        self.n = len(prompt)

    def feed(self, tok):
        self.kv, self.logits = self.orc.forward([tok], past_kv=self.kv, n_cached=self.n)
        self.n += 1


def _check(gpu_logits, ref_logits, gpu_tok, agree):
    err = rel_err(gpu_logits, ref_logits)
    assert err <= TOL, f"logits rel err {err:.3e}"
    abs_err = float((gpu_logits.float().cpu() - ref_logits).abs().max())
    if top1_margin(ref_logits) > 4 * abs_err:
        assert int(gpu_tok) == int(torch.argmax(ref_logits))
        agree.append(1)


@pytest.mark.parametrize("hbm", [False, True], ids=["host-tier", "hbm-tier"])
def test_greedy_decode_matches_oracle_teacher_forced(setup, hbm):
    spec, eng, orc, gen = setup
    free0 = eng.pool.free_blocks
    # 2 docs x 61 tokens + a 2-token query: the context crosses the 128-token block boundary while decoding
    reqs, prompts = zip(*[_request(spec, gen, eng, [4, 8], [61, 61], 3, 2, hbm),
                          _request(spec, gen, eng, [9], [200], 5, 9, hbm)])
    n_new = 12
    seqs = decode.start(eng, list(reqs), n_new)
    oracles = [_Oracle(orc, p) for p in prompts]
    logits0 = None
    agree = []
    try:
        # first token (prefill) vs the oracle's prompt logits
        for s, o in zip(seqs, oracles):
            if top1_margin(o.logits) > 0.5:
                assert s.tokens[0] == int(torch.argmax(o.logits))
        for t in range(1, n_new):
            for s, o in zip(seqs, oracles):
                o.feed(s.last)
            decode.step(eng, seqs)
            logits0 = eng._decode_step.logits[: len(seqs)].float().cpu()
            for i, (s, o) in enumerate(zip(seqs, oracles)):
                _check(logits0[i], o.logits, s.tokens[-1], agree)
        assert all(len(s.tokens) == n_new for s in seqs)
        assert len(agree) >= len(seqs) * (n_new - 1) // 4, f"argmax asserted on only {len(agree)} steps"
    finally:
        for s in seqs:
            decode.retire(eng, s)
        eng.resident.clear()
    assert eng.pool.free_blocks == free0


def test_continuous_batching_join_and_leave(setup):
    spec, eng, orc, gen = setup
    free0 = eng.pool.free_blocks
    specs = [([1, 2], [64, 64], 11, 16, 5), ([3], [130], 12, 7, 9), ([6, 7], [100, 28], 13, 30, 4),
             ([8], [64], 14, 1, 6)]
    cb = decode.ContinuousBatcher(eng, max_batch=2)
    ids, prompts = {}, {}
    for docs, ntok, qid, ql, mx in specs:
        req, prompt = _request(spec, gen, eng, docs, ntok, qid, ql, hbm=(qid % 2 == 0))
        rid = cb.submit(req, mx)
        ids[rid], prompts[rid] = mx, prompt
    out = cb.run()
    assert sorted(out) == sorted(ids)
    assert cb.prefills >= 2  # requests joined a running batch
    for rid, toks in out.items():
        assert len(toks) == ids[rid]
        # teacher-forced oracle: every generated token is the oracle's argmax where the margin is clear
        o = _Oracle(orc, prompts[rid])
        for k, tok in enumerate(toks):
            if k > 0:
                o.feed(toks[k - 1])
            if top1_margin(o.logits) > 0.05 * float(o.logits.abs().max()):
                assert tok == int(torch.argmax(o.logits)), f"request {rid} token {k}"
    cb.close()
    eng.resident.clear()
    assert eng.pool.free_blocks == free0


def test_decode_time_per_token_calibrates_cost_model(setup):
    from paper_2504_11765_b200.costs import CostParams

    spec, eng, orc, gen = setup
    free0 = eng.pool.free_blocks
    reqs = [_request(spec, gen, eng, [20 + i], [96], 30 + i, 8, hbm=False)[0] for i in range(4)]
    m = decode.decode_time_per_token(eng, reqs, n_steps=8)
    assert m["batch"] == 4 and m["seconds_per_step"] > 0 and m["tokens_per_s"] > 0
    p = CostParams(model=spec.profile(), decode_enabled=True, decode_time_per_token=m["seconds_per_token"])
    assert p.decode_time_per_token > 0
    assert eng.pool.free_blocks == free0
