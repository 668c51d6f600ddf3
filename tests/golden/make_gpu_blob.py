"""Fixture: a REAL document-KV blob written by the GPU path, for the CPU-side
cross-check that the reference's own KvStore reads what the B200 generator writes
(tests/test_gpu_fixture.py).  Run on a GPU box:

    python tests/golden/make_gpu_blob.py [out_dir]     # default tests/golden/gpu_store

Tiny model (configs[0] shape), weights = init_weights(seed 0) made on the CPU (so the
CPU test can rebuild them bit for bit) and copied to the GPU; the ordered combination
(3, 8) of 128 + 96 tokens is prefilled by librdkv (KvGenerator.generate: QKV epilogue
writes the .rdkv layout, FNV-1a on the GPU) and put through this package's KvStore into
tests/golden/gpu_store/ (blob file + manifest), exactly as a serving instance would.
"""
import json
import shutil
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import torch  # noqa: E402

from paper_2504_11765_b200.engine import Engine  # noqa: E402
from paper_2504_11765_b200.generator import KvGenerator  # noqa: E402
from paper_2504_11765_b200.model import get_spec, init_weights  # noqa: E402
from paper_2504_11765_b200.store import KvKey, KvStore  # noqa: E402

spec = get_spec("tiny")
w = init_weights(spec, 0, device="cpu").to("cuda")
eng = Engine(spec, weights=w, pool_tokens=4096)
gen = KvGenerator(eng, keep_on_device=False)
ids, counts = (3, 8), (128, 96)
blob = gen.generate(ids, counts)
torch.cuda.synchronize()
out = Path(sys.argv[1]) if len(sys.argv) > 1 else HERE / "gpu_store"
with tempfile.TemporaryDirectory() as tmp:
    st = KvStore(tmp)
    key = KvKey(spec.profile().model_hash, ids)
    st.put(key, blob)
    shutil.rmtree(out, ignore_errors=True)
    shutil.copytree(tmp, out)
(out / "fixture.json").write_text(json.dumps({
    "model": "tiny", "seed": 0, "doc_ids": list(ids), "doc_tokens": list(counts),
    "model_hash": spec.profile().model_hash, "checksum": blob.header.checksum,
    "gpu": torch.cuda.get_device_name(0)}, indent=1))
print("wrote", sorted(p.name for p in out.rglob("*")))
