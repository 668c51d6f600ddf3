"""Break a cold-disk TTFT (page cache dropped) into its parts: pinned-buffer allocation,
the parallel read, the GPU checksum, and the prefill.
    python scripts/micro/cold_path.py [model (llama-3.2-1b)] [docs (5)]   # C3: llama-3-8b 10"""
import json, sys, tempfile, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch
from paper_2504_11765_b200 import _lib
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.generator import KvGenerator
from paper_2504_11765_b200.model import get_spec, query_tokens
from paper_2504_11765_b200.prefill import PrefillRequest, prefill_batch
from paper_2504_11765_b200.store import GpuVerifier, KvKey, KvStore, read_blob_file

spec = get_spec(sys.argv[1] if len(sys.argv) > 1 else "llama-3.2-1b")
nd = int(sys.argv[2]) if len(sys.argv) > 2 else 5
eng = Engine(spec, seed=0, pool_tokens=16384, device_cache_bytes=1 << 30)
gen = KvGenerator(eng)
docs = tuple(11 * (i + 1) for i in range(nd))
blob = gen.generate(docs, (512,) * nd)
root = Path(tempfile.mkdtemp(prefix="rdkv_cold_"))
store = KvStore(root, 0, verifier=GpuVerifier("cuda"))
key = KvKey(spec.profile().model_hash, docs)
store.put(key, blob)
path = store.path_of(key)
L = _lib.lib()
qt = query_tokens(3, 64, spec.vocab)
rows = []
# "distinct": like the bench's cold leg, four freshly written composites, flushed, each read once
distinct = len(sys.argv) > 3 and sys.argv[3] == "distinct"
paths = [path]
if distinct:
    import os
    keys = [KvKey(spec.profile().model_hash, tuple(d + 1000 * j for d in docs)) for j in range(1, 5)]
    for k2 in keys:
        store.put(k2, gen.generate(k2.doc_ids, (512,) * nd))
    os.sync()
    paths = [store.path_of(k2) for k2 in keys]
for it in range(8):
    if distinct:
        key = keys[it % 4]
        path = paths[it % 4]
    L.rdkv_drop_page_cache(str(path).encode())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b2, _ = read_blob_file(path, verify=False)
    t1 = time.perf_counter()
    dev = GpuVerifier("cuda")(b2.payload, b2.header.checksum)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    L.rdkv_drop_page_cache(str(path).encode())
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    look = store.get(key)
    r = prefill_batch(eng, [PrefillRequest(look, None, qt, None)], timed=False)
    int(r.next_token[0])
    t4 = time.perf_counter()
    x = torch.empty(blob.header.payload_len, dtype=torch.uint8, pin_memory=True)
    t5 = time.perf_counter()
    del x
    rows.append({"read_ms": (t1 - t0) * 1e3, "gpu_verify_ms": (t2 - t1) * 1e3, "cold_ttft_ms": (t4 - t3) * 1e3,
                 "pinned_alloc_ms": (t5 - t4) * 1e3})
print(json.dumps({"payload_MiB": blob.header.payload_len / 2**20,
                  "median": {k: float(np.median([r[k] for r in rows])) for k in rows[0]}, "runs": rows}))
