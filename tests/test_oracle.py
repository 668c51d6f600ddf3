"""Pin the CPU oracle against the reference's own golden vectors before trusting it."""

import json
from pathlib import Path

from oracle import codec_ref
from oracle.store_ref import StoreModel

G = Path(__file__).resolve().parent / "golden"
CODEC = json.loads((G / "codec_golden.json").read_text())


def test_oracle_fnv_known_vectors():
    # reference test_codec.py:195-199
    assert codec_ref.fnv1a64(b"") == 0xCBF29CE484222325
    assert codec_ref.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert codec_ref.fnv1a64(b"foobar") == 0x85944171F73967E8
    for v in CODEC["fnv"]:
        assert "%016x" % codec_ref.fnv1a64(bytes.fromhex(v["hex"])) == v["hash"]
    for v in CODEC["fnv_seeded"]:
        assert "%016x" % codec_ref.fnv1a64(bytes.fromhex(v["hex"]), int(v["seed"], 16)) == v["hash"]


def test_oracle_reproduces_golden_hex():
    # reference test_codec.py:25-34: encode(synth_blob(ModelProfile('golden',2,8,2,4,2),[7,3,11],3,seed=99))
    enc = codec_ref.synth_encoded(("golden", 2, 8, 2, 4, 2), [7, 3, 11], 3, 99)
    assert enc.hex() == CODEC["golden_hex"]


def test_oracle_reproduces_reference_synth_blobs():
    for b in CODEC["synth_blobs"]:
        enc = codec_ref.synth_encoded(tuple(b["profile"]), b["doc_ids"], b["token_count"], b["seed"])
        assert enc.hex() == b["encoded_hex"]
        assert "%016x" % codec_ref.model_hash(*b["profile"]) == b["model_hash"]


def test_oracle_model_hashes_of_build_profiles():
    for p in CODEC["profiles"]:
        mh = codec_ref.model_hash(p["model_id"], p["layers"], p["kv_heads"] * p["head_dim"], p["kv_heads"],
                                  p["head_dim"], 2)
        assert "%016x" % mh == p["model_hash"]


def test_store_model_replays_reference_oplog():
    log = json.loads((G / "store_oplog.json").read_text())
    m = StoreModel(log["initial_capacity"])
    sizes = {}
    for op in log["ops"]:
        key = tuple(op["doc_ids"])
        size = 16 + 8 * len(key) + 30 + 2 * 1 * 1 * 4 * op["tokens"] * 2
        if op["op"] == "put":
            # checksum stands in for content identity: seed 0 vs 1
            got = m.put(key, size, op["seed"] if key not in m.disk else op["seed"])
            if key in sizes and sizes[key] != op["seed"]:
                got = "ImmutableEntryError"
            sizes.setdefault(key, op["seed"])
            assert got == op["result"], op
        elif op["op"] == "get":
            outcome, cost = m.get(key)
            assert (outcome, cost) == (op["result"], op["load_cost_bytes"]), op
        elif op["op"] == "contains":
            assert m.contains(key) == op["result"], op
        else:
            m.set_capacity(op["capacity"])
        assert m.stats == op["stats"], op
