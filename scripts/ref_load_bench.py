"""SURVEY §8(d) CPU timing plan, item 1: the reference's own load path
(`ragdcache.KvStore.get`, disk hit = read + decode + pure-Python FNV verify)
timed with perf_counter against files written by this package's store, next to
this package's host load path on the same files.  Runs where /root/reference is
mounted (this container); the GPU box has no reference.

    python scripts/ref_load_bench.py > profiles/r1_ref_load_path.json
"""
import importlib
import json
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_11765_b200 import _lib  # noqa: E402
from paper_2504_11765_b200.codec import synth_blob  # noqa: E402
from paper_2504_11765_b200.model import get_spec  # noqa: E402
from paper_2504_11765_b200.store import KvKey, KvStore, Outcome  # noqa: E402

REF = Path("/root/reference/pkg/src")


def main():
    spec = get_spec("llama-3.2-1b")
    prof = spec.profile()
    docs, tokens = (101,), 512  # one C2 document: 16 MiB payload
    blob = synth_blob(prof, docs, tokens)
    root = Path(tempfile.mkdtemp(prefix="rdkv_refload_"))
    ours = KvStore(root, 0)
    key = KvKey(prof.model_hash, docs)
    ours.put(key, blob)
    path = ours.path_of(key)
    size = path.stat().st_size
    out = {"config": "C2 single document (512 tokens, llama-3.2-1b-shaped), file written by this package",
           "file_bytes": size, "host_cores": os.cpu_count()}

    def timed(fn, reps):
        ts = []
        for _ in range(reps):
            _lib.lib().rdkv_drop_page_cache(str(path).encode())
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    # this package: aligned parallel read + native FNV verify (host path, no GPU here)
    t = timed(lambda: KvStore(root, 0).get(key), 3)
    out["ours_host_get_s"] = t
    out["ours_host_get_MBps"] = size / t / 1e6
    if (REF / "ragdcache").exists():
        sys.path.insert(0, str(REF))
        rstore = importlib.import_module("ragdcache.store")
        rk = rstore.KvKey(prof.model_hash, docs)

        def ref_get():
            look = rstore.KvStore(root, 0).get(rk)  # recovers the index from manifest.jsonl
            assert look.outcome.name == "DISK_HIT", look.outcome
            assert bytes(look.blob.payload) == blob.payload_bytes()

        t = timed(ref_get, 1)
        out["reference_get_s"] = t
        out["reference_get_MBps"] = size / t / 1e6
        out["speedup_host"] = out["reference_get_s"] / out["ours_host_get_s"]
    else:
        out["reference_get_s"] = None
    assert KvStore(root, 0).get(key).outcome is Outcome.DISK_HIT
    print(json.dumps(out))


if __name__ == "__main__":
    main()
