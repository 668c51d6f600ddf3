"""paper_2504_11765_b200.codec vs the reference's golden bytes (bit-exact)."""

import json
from pathlib import Path

import pytest
import torch
from hypothesis import given, settings, strategies as st

from paper_2504_11765_b200 import codec
from paper_2504_11765_b200.codec import (BadMagicError, ChecksumMismatchError, KvBlob, MalformedHeaderError,
                                         ModelProfile, TruncatedError, UnsupportedVersionError, decode, encode,
                                         fnv1a64, synth_blob)
from paper_2504_11765_b200.model import SPECS
from paper_2504_11765_b200.store import KvKey

G = json.loads((Path(__file__).resolve().parent / "golden" / "codec_golden.json").read_text())
ERR = {"BadMagicError": BadMagicError, "UnsupportedVersionError": UnsupportedVersionError,
       "TruncatedError": TruncatedError, "ChecksumMismatchError": ChecksumMismatchError,
       "MalformedHeaderError": MalformedHeaderError}


def test_fnv_vectors():
    for v in G["fnv"]:
        assert "%016x" % fnv1a64(bytes.fromhex(v["hex"])) == v["hash"]
    for v in G["fnv_seeded"]:
        assert "%016x" % fnv1a64(bytes.fromhex(v["hex"]), int(v["seed"], 16)) == v["hash"]


def test_fnv_many_matches_serial():
    bufs = [bytes.fromhex(v["hex"]) for v in G["fnv"]]
    assert codec.fnv1a64_many(bufs, threads=4) == [fnv1a64(b) for b in bufs]


def test_fnv_over_pinned_style_tensor():
    t = torch.arange(1000, dtype=torch.int32).view(torch.uint8)
    assert fnv1a64(t) == fnv1a64(t.numpy().tobytes())


def test_golden_hex_roundtrip():
    p = ModelProfile("golden", 2, 8, 2, 4, 2)
    b = synth_blob(p, [7, 3, 11], 3, seed=99)
    assert encode(b).hex() == G["golden_hex"]
    assert decode(bytes.fromhex(G["golden_hex"])) == b
    h = b.header
    assert h.model_hash == 0x5E99A4AB5BA66216 and h.checksum == 0x3EF65C21123369EB and h.payload_len == 192


def test_reference_synth_blobs_bit_exact():
    for g in G["synth_blobs"]:
        p = ModelProfile(*g["profile"])
        assert "%016x" % p.model_hash == g["model_hash"]
        b = synth_blob(p, g["doc_ids"], g["token_count"], seed=g["seed"])
        assert encode(b).hex() == g["encoded_hex"]
        assert decode(bytes.fromhex(g["encoded_hex"])) == b


def test_build_profiles_hash_like_reference():
    by_id = {p["model_id"]: p for p in G["profiles"]}
    for spec in (SPECS["tiny"], SPECS["llama-3.2-1b"], SPECS["llama-3-8b"], SPECS["llama-3-70b"]):
        prof = spec.profile()
        g = by_id[prof.model_id]
        assert "%016x" % prof.model_hash == g["model_hash"]
        assert codec.blob_size(prof, 512) == g["blob_size_512"]
        assert codec.encoded_size(prof, 2560, 5) == g["encoded_size_5x512"]


def test_key_paths():
    for k in G["keys"]:
        key = KvKey(0x5E99A4AB5BA66216, tuple(k["doc_ids"]))
        assert key.file_stem == k["file_stem"]


@pytest.mark.parametrize("case", G["decode_errors"], ids=lambda c: c["name"])
def test_decode_error_taxonomy(case):
    data = bytes.fromhex(case["hex"])
    if case["error"] is None:
        decode(data)
    else:
        with pytest.raises(ERR[case["error"]]):
            decode(data)


def test_profile_validation():
    with pytest.raises(ValueError):
        ModelProfile("bad", 2, 10, 2, 4)
    with pytest.raises(ValueError):
        ModelProfile("bad", 2, 8, 2, 4, elem_width=3)
    with pytest.raises(ValueError):
        synth_blob(ModelProfile("t", 1, 4, 1, 4), [], 2)


def test_blob_invariants_enforced():
    b = synth_blob(ModelProfile("t", 2, 8, 2, 4), [1, 2], 4, seed=3)
    with pytest.raises(ValueError):
        KvBlob(b.header, b.payload[:-1] + b"\x00")
    with pytest.raises(ValueError):
        KvBlob(b.header, b.payload[:-1])
    assert KvBlob(b.header, b.payload) == b


@given(st.integers(1, 4), st.integers(1, 4), st.integers(1, 8), st.sampled_from([2, 4]),
       st.lists(st.integers(0, 2 ** 64 - 1), min_size=1, max_size=6), st.integers(1, 16), st.integers(0, 2 ** 64 - 1))
@settings(max_examples=60, deadline=None)
def test_roundtrip_property(layers, kv, hd, ew, ids, n, seed):
    p = ModelProfile(f"m{layers}x{kv}x{hd}", layers, kv * hd, kv, hd, ew)
    b = synth_blob(p, ids, n, seed)
    enc = encode(b)
    assert len(enc) == codec.encoded_size(p, n, len(ids))
    out = decode(enc)
    assert out == b and encode(out) == enc
