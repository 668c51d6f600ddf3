"""Generate the golden fixtures of tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src; nothing is
copied.  The JSON files it writes are committed so the GPU box (which has no
/root/reference) can check parity against them.
"""

from __future__ import annotations

import json
import random
import shutil
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from ragdcache import codec, costs, prefetch, sim, store, workload  # noqa: E402
from ragdcache.service import SharedCacheService  # noqa: E402


def dump(name: str, obj) -> None:
    (HERE / name).write_text(json.dumps(obj, sort_keys=True, indent=1) + "\n")
    print("wrote", name)


# ----------------------------------------------------------------- codec
def make_codec() -> None:
    out: dict = {}
    golden_profile = codec.ModelProfile("golden", 2, 8, 2, 4, 2)
    out["golden_hex"] = codec.encode(codec.synth_blob(golden_profile, [7, 3, 11], 3, seed=99)).hex()
    rng = random.Random(1234)
    vec = [b"", b"a", b"foobar", bytes(range(256)), b"\x00" * 1000]
    vec += [bytes(rng.getrandbits(8) for _ in range(rng.randint(1, 300))) for _ in range(10)]
    out["fnv"] = [{"hex": v.hex(), "hash": "%016x" % codec.fnv1a64(v)} for v in vec]
    out["fnv_seeded"] = [{"hex": v.hex(), "seed": "%016x" % s, "hash": "%016x" % codec.fnv1a64(v, s)}
                         for v, s in [(b"abc", 0), (b"xyz", 12345), (b"hello world", 0xFFFFFFFFFFFFFFFF)]]
    blobs = []
    for i in range(12):
        kv, hd = rng.randint(1, 4), rng.randint(1, 8)
        p = codec.ModelProfile(f"m{i}", rng.randint(1, 3), kv * hd, kv, hd, rng.choice([2, 4]))
        ids = [rng.getrandbits(64) if i % 3 == 0 else rng.randint(0, 50) for _ in range(rng.randint(1, 5))]
        n = rng.randint(1, 6)
        seed = rng.getrandbits(64)
        b = codec.synth_blob(p, ids, n, seed=seed)
        blobs.append({"profile": [p.model_id, p.layers, p.hidden_dim, p.kv_heads, p.head_dim, p.elem_width],
                      "model_hash": "%016x" % p.model_hash, "doc_ids": ids, "token_count": n, "seed": seed,
                      "encoded_hex": codec.encode(b).hex()})
    out["synth_blobs"] = blobs
    # profiles of the model shapes the B200 build runs (SURVEY H-b: hidden := kv_heads*head_dim)
    shapes = {"tiny/bf16": (2, 4, 64), "llama-3.2-1b/bf16": (16, 8, 64), "llama-3-8b/bf16": (32, 8, 128),
              "llama-3-70b/bf16": (80, 8, 128)}
    out["profiles"] = []
    for mid, (L, kv, hd) in shapes.items():
        p = codec.ModelProfile(mid, L, kv * hd, kv, hd, 2)
        out["profiles"].append({"model_id": mid, "layers": L, "kv_heads": kv, "head_dim": hd,
                                "model_hash": "%016x" % p.model_hash,
                                "blob_size_512": codec.blob_size(p, 512),
                                "encoded_size_5x512": codec.encoded_size(p, 2560, 5)})
    keys = []
    for ids in ([1], [7, 3, 11], [2, 1], [1, 2], list(range(20)), [2 ** 64 - 1]):
        k = store.KvKey(0x5E99A4AB5BA66216, tuple(ids))
        keys.append({"doc_ids": ids, "file_stem": k.file_stem,
                     "rel_path": f"{k.model_hash:016x}/{k.file_stem}.rdkv"})
    out["keys"] = keys
    # decode error taxonomy (test_codec.py:149-192 cases + a few more)
    base = codec.encode(codec.synth_blob(codec.ModelProfile("tiny", 2, 8, 2, 4, 2), [1, 2], 4, seed=3))
    hl = codec.header_size(2)
    cases = {
        "bad_magic": b"XXXX" + base[4:],
        "bad_version": base[:4] + b"\x63\x00" + base[6:],
        "byte_flip": base[:hl] + bytes([base[hl] ^ 0xFF]) + base[hl + 1:],
        "truncated_payload": base[:-1],
        "truncated_header": base[:10],
        "trailing": base + b"\x00",
        "nonzero_reserved": base[: hl - 17] + b"\x01" + base[hl - 16:],
        "zero_docs": base[:14] + b"\x00\x00" + base[16:],
        "bad_payload_len": base[: hl - 16] + (999).to_bytes(8, "little") + base[hl - 8:],
        "empty": b"",
    }
    errs = []
    for name, data in cases.items():
        try:
            codec.decode(data)
            cls = None
        except codec.CodecError as exc:
            cls = type(exc).__name__
        errs.append({"name": name, "hex": data.hex(), "error": cls})
    out["decode_errors"] = errs
    dump("codec_golden.json", out)


# ----------------------------------------------------------------- store op log
def make_store() -> None:
    prof = codec.ModelProfile("tiny", 1, 4, 1, 4, 2)
    rng = random.Random(77)
    tmp = Path(tempfile.mkdtemp())
    try:
        entry = codec.synth_blob(prof, [1], 2).header.encoded_size
        st = store.KvStore(tmp / "s", memory_capacity_bytes=3 * entry + 10)
        ops = []
        for i in range(400):
            r = rng.random()
            ids = tuple(rng.sample(range(1, 9), rng.randint(1, 2)))
            tokens = 1 + (sum(ids) % 3)
            key = store.KvKey(prof.model_hash, ids)
            rec = {"i": i, "doc_ids": list(ids), "tokens": tokens}
            if r < 0.35:
                rec["op"] = "put"
                seed = 0 if rng.random() < 0.9 else 1
                rec["seed"] = seed
                try:
                    st.put(key, codec.synth_blob(prof, ids, tokens, seed=seed))
                    rec["result"] = "ok"
                except store.StoreError as exc:
                    rec["result"] = type(exc).__name__
            elif r < 0.8:
                rec["op"] = "get"
                res = st.get(key)
                rec["result"] = res.outcome.value
                rec["load_cost_bytes"] = res.load_cost_bytes
                rec["checksum"] = "%016x" % res.blob.header.checksum if res.blob else None
            elif r < 0.95:
                rec["op"] = "contains"
                rec["result"] = st.contains(key).value
            else:
                rec["op"] = "set_capacity"
                cap = rng.choice([0, entry, 2 * entry + 5, 3 * entry + 10, 10 * entry])
                rec["capacity"] = cap
                st.set_memory_capacity(cap)
                rec["result"] = "ok"
            rec["stats"] = json.loads(st.stats().to_json())
            ops.append(rec)
        reopened = store.KvStore(tmp / "s", memory_capacity_bytes=0)
        recovered = sorted([list(k.doc_ids) for k in reopened.keys()])
        manifest = (tmp / "s" / "manifest.jsonl").read_text().splitlines()
        dump("store_oplog.json", {"profile": ["tiny", 1, 4, 1, 4, 2], "initial_capacity": 3 * entry + 10,
                                  "ops": ops, "recovered_keys": recovered,
                                  "recovered_stats": json.loads(reopened.stats().to_json()),
                                  "manifest": manifest})
    finally:
        shutil.rmtree(tmp)


# ----------------------------------------------------------------- workload / costs / prefetch
def make_workload() -> None:
    out = {}
    for (n, s, q, seed, k) in [(50, 1.0, 12, 3, 2), (10000, 1.0, 64, 1, 10), (1000, 0.9609375, 100, 7, 1),
                               (20, 0.5, 30, 11, 5)]:
        items = workload.zipf_stream(n, s, q, seed=seed, k=k, q_tokens=64, doc_tokens=512)
        out[f"zipf_{n}_{s}_{q}_{seed}_{k}"] = [list(it.doc_ids) for it in items]
    items = workload.zipf_stream(50, 1.0, 20, seed=3)
    out["poisson_40_seed9"] = [t for t, _ in workload.poissonize(items, 40.0, seed=9)]
    out["uniform_100"] = [t for t, _ in workload.uniform_arrivals(items, 100.0)]
    dump("workload_golden.json", out)


def make_costs_prefetch() -> None:
    out = {"prefill_work": [], "cached_prefill_work": [], "plan_tasks": []}
    for L, D, n in [(24, 2048, 128), (16, 512, 2624), (32, 1024, 5184), (2, 8, 0)]:
        out["prefill_work"].append([L, D, n, costs.prefill_work(L, D, n)])
    for L, D, q, c in [(24, 2048, 16, 120), (16, 512, 64, 2560), (32, 1024, 64, 5120)]:
        out["cached_prefill_work"].append([L, D, q, c, costs.cached_prefill_work(L, D, q, c)])
    prof = codec.ModelProfile("tiny", 1, 4, 1, 4, 2)
    tmp = Path(tempfile.mkdtemp())
    try:
        svc = SharedCacheService(store.KvStore(tmp, memory_capacity_bytes=0))
        svc.put(store.KvKey(prof.model_hash, (4,)), codec.synth_blob(prof, [4], 10))
        for qid, ids, toks in [(0, (4, 2, 9), (10, 20, 30)), (1, (1, 2), (5, 6)), (2, (4,), (10,))]:
            pq = prefetch.PendingQuery(qid, 0.0, len(ids), 8, doc_ids=ids, doc_tokens=toks)
            tasks = prefetch.plan_tasks(pq, prof, svc, None)
            out["plan_tasks"].append({"doc_ids": list(ids), "doc_tokens": list(toks),
                                      "tasks": [[list(t.key.doc_ids), t.est_work] for t in tasks]})
    finally:
        shutil.rmtree(tmp)
    dump("costs_prefetch_golden.json", out)


# ----------------------------------------------------------------- scheduler
def make_sim() -> None:
    shutil.copy(Path("/root/reference/pkg/tests/golden/sim_small_report.json"), HERE / "sim_small_report.json")
    print("copied sim_small_report.json (reference golden)")
    MODEL = codec.ModelProfile("sim-tiny", layers=2, hidden_dim=8, kv_heads=2, head_dim=4, elem_width=2)
    PARAMS = costs.CostParams(model=MODEL, network_delay=0.001)
    RATE = 1.0e7
    gpu = lambda name: costs.DeviceProfile(name, costs.DeviceKind.INFERENCE_GPU, RATE)
    devs = {
        "baseline": (gpu("gpu0"), gpu("gpu1")),
        "a": (gpu("gpu0"), costs.DeviceProfile("gen0", costs.DeviceKind.GENERATOR_GPU, RATE * 0.5)),
        "b": (gpu("gpu0"), gpu("gpu1"), costs.DeviceProfile("cpu0", costs.DeviceKind.CPU, RATE * 0.1)),
    }
    runs = {}
    cases = [("baseline", "poisson", 1, 1, 40.0, 1024), ("a", "poisson", 2, 3, 60.0, 0),
             ("b", "uniform", 3, 2, 80.0, 50000), ("a", "uniform", 1, 3, 200.0, 3000)]
    for cfgname, proc, k, tries, rate, mem in cases:
        cfg = sim.SimConfig(configuration=costs.Configuration(cfgname), devices=devs[cfgname], cost=PARAMS,
                            arrival=sim.ArrivalSpec(rate=rate, process=sim.ArrivalProcess(proc)), k=k, tries=tries,
                            seed=5, threshold=0.03, memory_capacity_bytes=mem)
        items = workload.zipf_stream(40, 1.0, 30, seed=2, k=k, q_tokens=16, doc_tokens=120)
        report, records = sim.run(cfg, items)
        runs[f"{cfgname}_{proc}_k{k}_t{tries}_r{rate}_m{mem}"] = {
            "report": report.to_dict(), "records": [r.to_dict() for r in records]}
    single = sim.SimConfig(configuration=costs.Configuration.SINGLE_INSTANCE, devices=(gpu("gpu0"),), cost=PARAMS,
                           arrival=sim.ArrivalSpec(rate=10.0), k=1, tries=1, seed=1, threshold=0.5,
                           memory_capacity_bytes=2000)
    items = workload.zipf_stream(40, 1.0, 25, seed=4, k=2, q_tokens=16, doc_tokens=120)
    for b in (1, 4):
        for use in (True, False):
            rep, recs = sim.run_single_instance(single, items, batch_size=b, use_cache=use)
            runs[f"single_b{b}_{use}"] = {"report": rep.to_dict(), "records": [r.to_dict() for r in recs]}
    cfg = sim.SimConfig(configuration=costs.Configuration.BASELINE, devices=devs["baseline"], cost=PARAMS,
                        arrival=sim.ArrivalSpec(rate=50.0), k=1, tries=1, seed=1, threshold=0.05)
    items = workload.zipf_stream(50, 1.0, 20, seed=1, k=1, q_tokens=16, doc_tokens=120)
    runs["sweep"] = [p.to_dict() for p in sim.sweep_rate(cfg, [5.0, 20.0, 80.0], items)]
    runs["capacity"] = sim.service_capacity(cfg, items)
    (HERE / "sim_runs.json").write_text(json.dumps(runs, sort_keys=True, indent=1) + "\n")
    print("wrote sim_runs.json")


if __name__ == "__main__":
    make_codec()
    make_store()
    make_workload()
    make_costs_prefetch()
    make_sim()
