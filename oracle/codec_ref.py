"""Python side of the codec oracle (TEST INFRASTRUCTURE; see oracle/__init__.py).

`load()` binds oracle/_build/libcodec_ref.so (built by oracle/Makefile from
codec_ref.c).  `synth_encoded()` rebuilds a reference `.rdkv` encoding from the
C restatement alone, following codec.synth_blob + codec.encode
(codec.py:188-239), so tests can check byte-for-byte against the goldens the
reference produced.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "_build" / "libcodec_ref.so"
_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


def load():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build()
        L = C.CDLL(str(_SO))
        u64, vp = C.c_uint64, C.c_void_p
        L.oracle_fnv1a64.restype, L.oracle_fnv1a64.argtypes = u64, [C.c_char_p, u64, u64]
        L.oracle_fnv_offset.restype = u64
        L.oracle_splitmix64.restype, L.oracle_splitmix64.argtypes = u64, [u64]
        L.oracle_synth_state.restype = u64
        L.oracle_synth_state.argtypes = [u64, u64, C.POINTER(u64), u64, u64]
        L.oracle_keystream.restype, L.oracle_keystream.argtypes = None, [u64, vp, u64]
        L.oracle_encode_header.restype = u64
        L.oracle_encode_header.argtypes = [vp, u64, C.POINTER(u64), C.c_uint16, C.c_uint32, C.c_uint16,
                                           C.c_uint16, C.c_uint16, C.c_uint8, u64, u64]
        _lib = L
    return _lib


def fnv1a64(data: bytes, seed: int | None = None) -> int:
    L = load()
    return int(L.oracle_fnv1a64(data, len(data), L.oracle_fnv_offset() if seed is None else seed))


def model_hash(model_id: str, layers: int, hidden: int, kv_heads: int, head_dim: int, elem_width: int) -> int:
    """ModelProfile.model_hash (codec.py:95-107)."""
    s = "\x00".join(str(x) for x in (model_id, layers, hidden, kv_heads, head_dim, elem_width))
    return fnv1a64(s.encode("utf-8"))


def synth_encoded(profile, doc_ids, token_count: int, seed: int) -> bytes:
    """encode(synth_blob(...)) from the C restatement only."""
    L = load()
    mid, layers, hidden, kvh, hd, ew = profile
    mh = model_hash(mid, layers, hidden, kvh, hd, ew)
    ids = (C.c_uint64 * len(doc_ids))(*doc_ids)
    state = L.oracle_synth_state(seed, mh, ids, len(doc_ids), token_count)
    n = 2 * layers * kvh * hd * token_count * ew
    payload = C.create_string_buffer(max(n, 1))
    L.oracle_keystream(state, payload, n)
    body = payload.raw[:n]
    head = C.create_string_buffer(46 + 8 * len(doc_ids))
    hl = L.oracle_encode_header(head, mh, ids, len(doc_ids), token_count, layers, kvh, hd, ew, n,
                                fnv1a64(body))
    return head.raw[:hl] + body
