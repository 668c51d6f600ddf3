"""Logits of one 16-query C2-shaped batch (M = 1024 query rows over a 5 x 512 composite in
the HBM tier) -> argv[1] (.npy).  tests/test_gemm_sk_gpu.py runs it under each
RDKV_GEMM_SK mode (read once per process) and compares the modes."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import KvKey, LookupResult, Outcome

spec = get_spec("llama-3.2-1b")
eng = Engine(spec, seed=0, pool_tokens=4096, device_cache_bytes=spec.kv_bytes_per_token() * 2600)
gen = KvGenerator(eng, keep_on_device=True)
docs = (4211, 17, 905, 3, 77)
blob = gen.generate(docs, (512,) * 5)
key = KvKey(spec.profile().model_hash, docs)
reqs = [PrefillRequest(LookupResult(Outcome.MEMORY_HIT, blob, 0), None, query_tokens(100 + i, 64, spec.vocab), key)
        for i in range(16)]
r = prefill_batch(eng, reqs, timed=False)
torch.cuda.synchronize()
np.save(sys.argv[1], r.logits.float().cpu().numpy())
