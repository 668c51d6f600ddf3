"""C1 (tiny) hot path for compute-sanitizer: document-KV generation, blob put/get
through the store, host-tier load (H2D + K3 unpack), cached-prefix prefill,
full-prompt prefill, the GPU FNV-1a, and the decode phase (greedy steps across a
pool-block boundary, a chunked-prefill extend).  Run as
    compute-sanitizer --tool memcheck python scripts/sanitize_c1.py"""
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2504_11765_b200 import decode
from paper_2504_11765_b200.codec import fnv1a64, fnv1a64_device
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import KvKey, KvStore, LookupResult, Outcome

spec = get_spec("tiny")
eng = Engine(spec, seed=0, pool_tokens=4096, device_cache_bytes=8 << 20)
gen = KvGenerator(eng, keep_on_device=True)
docs, counts = (3, 8, 5), (128, 96, 128)
with tempfile.TemporaryDirectory() as root:
    store = KvStore(root, memory_capacity_bytes=64 << 20)
    key = KvKey(spec.profile().model_hash, docs)
    store.put(key, gen.generate(docs, counts))
    look = store.get(key)
    q = query_tokens(1, 32, spec.vocab)
    r1 = prefill_batch(eng, [PrefillRequest(look, None, q, None)], timed=False)       # host tier: H2D + K3
    r2 = prefill_batch(eng, [PrefillRequest(look, None, q, key)], timed=False, use_graph=False)  # HBM tier
    r3 = prefill_batch(eng, [PrefillRequest(LookupResult(Outcome.MISS), gen.tokens(docs, counts), q)],
                       timed=False, use_graph=False)                                  # full prompt
    raw = torch.from_numpy(np.frombuffer(bytes(look.blob.payload_tensor().numpy()), np.uint8).copy()).cuda()
    assert fnv1a64_device(raw) == fnv1a64(bytes(look.blob.payload_tensor().numpy()))
    # decode: both sequences' contexts end on a block boundary (352 + 32 = 6 x 64), so the
    # first step opens a new pool block; then a 70-token chunk spans two more blocks
    seqs = decode.start(eng, [PrefillRequest(look, None, q, key), PrefillRequest(look, None, q, None)], 6)
    while any(not s.done for s in seqs):
        decode.step(eng, seqs)
    assert seqs[0].tokens == seqs[1].tokens, (seqs[0].tokens, seqs[1].tokens)
    nxt = decode.extend(eng, [(seqs[0].live, query_tokens(2, 70, spec.vocab))])
    for s in seqs:
        decode.retire(eng, s)
    torch.cuda.synchronize()
    print("decode", seqs[0].tokens, int(nxt[0]))
    print("tokens", int(r1.next_token[0]), int(r2.next_token[0]), int(r3.next_token[0]))
