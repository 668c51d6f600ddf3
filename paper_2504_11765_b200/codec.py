"""`.rdkv` KV-blob format — drop-in for ``ragdcache.codec`` (reference codec.py:1-295).

The layout (all little-endian) is the reference's, bit for bit (codec.py:8-13):

    magic "RDKV" | version u16 | model_hash u64 | doc_count u16 | doc_ids u64*k
    | token_count u32 | layers u16 | kv_heads u16 | head_dim u16 | elem_width u8
    | reserved 3x0 | payload_len u64 | checksum u64 | payload

Header (de)serialisation and the FNV-1a checksum run in librdkv (H1,
``include/rdkv.h``).  What changes on B200 is the *payload*: instead of the
splitmix64 noise of ``synth_blob`` (codec.py:188-224) it holds real document KV
written by the document-prefill kernels, laid out head-major as
``[layers][2 (K,V)][kv_heads][token_count][head_dim]`` bf16 with K post-RoPE at
positions 0..token_count-1.  A payload may be ``bytes`` (the
reference type) or a CPU ``torch.Tensor`` of uint8 backed by pinned memory, so
the memory tier can DMA straight into HBM.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib

MAGIC = b"RDKV"
VERSION = 1
FNV_OFFSET = 0xCBF29CE484222325
_U64 = (1 << 64) - 1


class CodecError(Exception):
    """Base class for blob encode/decode failures (codec.py:40)."""


class BadMagicError(CodecError):
    pass


class UnsupportedVersionError(CodecError):
    pass


class TruncatedError(CodecError):
    pass


class ChecksumMismatchError(CodecError):
    pass


class MalformedHeaderError(CodecError):
    pass


_ERR_CLASS = {
    _lib.RDKV_ERR_BAD_MAGIC: BadMagicError,
    _lib.RDKV_ERR_UNSUPPORTED_VERSION: UnsupportedVersionError,
    _lib.RDKV_ERR_TRUNCATED: TruncatedError,
    _lib.RDKV_ERR_CHECKSUM: ChecksumMismatchError,
    _lib.RDKV_ERR_MALFORMED: MalformedHeaderError,
}


def raise_for(rc: int) -> None:
    """Translate a librdkv status into the reference exception class."""
    if rc >= 0:
        return
    cls = _ERR_CLASS.get(rc)
    if cls is None:
        raise _lib.NativeError(rc, _lib.last_error())
    raise cls(_lib.last_error())


# ----------------------------------------------------------------- buffers


def buffer_address(buf) -> tuple[int, int]:
    """(address, nbytes) of a bytes-like object or a contiguous CPU uint8 tensor."""
    if hasattr(buf, "data_ptr"):
        return int(buf.data_ptr()), int(buf.numel() * buf.element_size())
    arr = np.frombuffer(buf, dtype=np.uint8)
    return (int(arr.ctypes.data) if arr.size else 0), int(arr.size)


def as_bytes(buf) -> bytes:
    if isinstance(buf, bytes):
        return buf
    if hasattr(buf, "data_ptr"):
        return buf.contiguous().numpy().tobytes()
    return bytes(buf)


def fnv1a64(data, seed: int = FNV_OFFSET) -> int:
    """64-bit FNV-1a (codec.py:64-69), computed natively."""
    addr, n = buffer_address(data)
    return int(_lib.lib().rdkv_fnv1a64(addr, n, seed & _U64))


def fnv1a64_device(data, seed: int = FNV_OFFSET, stream=None) -> int:
    """64-bit FNV-1a of a CUDA uint8 tensor, computed on its GPU (rdkv_fnv1a64_device:
    low-byte automaton + affine chunk composition, bit-exact with codec.py:64-69)."""
    import torch

    if not (hasattr(data, "is_cuda") and data.is_cuda):
        raise TypeError("fnv1a64_device needs a CUDA tensor")
    L = _lib.lib()
    raw = data.reshape(-1).view(torch.uint8) if data.dtype != torch.uint8 else data.reshape(-1)
    n = raw.numel()
    need = int(L.rdkv_fnv1a64_device_scratch(n))
    ws = torch.empty(need, dtype=torch.uint8, device=raw.device)
    out = torch.empty(1, dtype=torch.int64, device=raw.device)
    st = stream if stream is not None else torch.cuda.current_stream(raw.device)
    _lib.check(L.rdkv_fnv1a64_device(raw.data_ptr(), n, seed & _U64, ws.data_ptr(), need, out.data_ptr(),
                                     st.cuda_stream))
    st.synchronize()
    return int(out.item()) & _U64


def fnv1a64_device_async(data, seed: int = FNV_OFFSET, stream=None):
    """fnv1a64_device without the host synchronisation: returns a 1-element int64 CUDA
    tensor that holds the checksum once ``stream`` reaches this point."""
    import torch

    L = _lib.lib()
    raw = data.reshape(-1).view(torch.uint8) if data.dtype != torch.uint8 else data.reshape(-1)
    n = raw.numel()
    need = int(L.rdkv_fnv1a64_device_scratch(n))
    st = stream if stream is not None else torch.cuda.current_stream(raw.device)
    with torch.cuda.stream(st):
        ws = torch.empty(need, dtype=torch.uint8, device=raw.device)
        out = torch.empty(1, dtype=torch.int64, device=raw.device)
    _lib.check(L.rdkv_fnv1a64_device(raw.data_ptr(), n, seed & _U64, ws.data_ptr(), need, out.data_ptr(),
                                     st.cuda_stream))
    return out


class StreamingFnv:
    """Device FNV-1a of a CUDA uint8 buffer that fills front to back (a streamed disk
    hit): ``advance(ready)`` runs the per-chunk automaton pass over the newly complete
    16-KiB chunks on ``stream``; ``result()`` runs the rest and returns the checksum —
    equal to fnv1a64_device of the whole buffer."""

    def __init__(self, data, seed: int = FNV_OFFSET, stream=None) -> None:
        import torch

        self.raw = data.reshape(-1)
        self.n = self.raw.numel()
        self.seed = seed & _U64
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.raw.device)
        L = _lib.lib()
        self.need = int(L.rdkv_fnv1a64_device_scratch(self.n))
        with torch.cuda.stream(self.stream):
            self.ws = torch.empty(self.need, dtype=torch.uint8, device=self.raw.device)
            self.out = torch.empty(1, dtype=torch.int64, device=self.raw.device)
        self.next = 0

    def advance(self, ready: int) -> None:
        c = int(_lib.lib().rdkv_fnv1a64_device_partial(self.raw.data_ptr(), self.n, min(ready, self.n), self.next,
                                                       self.ws.data_ptr(), self.need, self.stream.cuda_stream))
        _lib.check(c)
        self.next = c

    def result(self) -> int:
        self.advance(self.n)
        L = _lib.lib()
        _lib.check(L.rdkv_fnv1a64_device_finish(self.raw.data_ptr(), self.n, self.seed, self.ws.data_ptr(), self.need,
                                                self.out.data_ptr(), self.stream.cuda_stream))
        self.stream.synchronize()
        return int(self.out.item()) & _U64


def fnv1a64_many(buffers: Sequence, threads: int = 8) -> list[int]:
    """FNV-1a of several independent buffers in parallel (one chain per buffer)."""
    n = len(buffers)
    if n == 0:
        return []
    addrs = (C.c_void_p * n)()
    lens = (C.c_size_t * n)()
    for i, b in enumerate(buffers):
        addrs[i], lens[i] = buffer_address(b)
    out = (C.c_uint64 * n)()
    _lib.lib().rdkv_fnv1a64_many(addrs, lens, n, out, threads)
    return [int(x) for x in out]


# ----------------------------------------------------------------- profile


@dataclass(frozen=True)
class ModelProfile:
    """Dimensions that fix the KV-cache size of one model (codec.py:72-107).

    The reference requires ``kv_heads * head_dim == hidden_dim`` (codec.py:89-93),
    which grouped-query models violate; GQA models are described with
    ``hidden_dim := kv_heads * head_dim`` and carry their real name and dtype in
    ``model_id`` (see :func:`profile_for`), so the reference's own code computes
    identical sizes, headers and hashes.
    """

    model_id: str
    layers: int
    hidden_dim: int
    kv_heads: int
    head_dim: int
    elem_width: int = 2

    def __post_init__(self) -> None:
        for attr in ("layers", "hidden_dim", "kv_heads", "head_dim"):
            if getattr(self, attr) < 1:
                raise ValueError(f"{attr} must be >= 1")
        if self.elem_width not in (2, 4):
            raise ValueError("elem_width must be 2 or 4 bytes")
        if self.kv_heads * self.head_dim != self.hidden_dim:
            raise ValueError(
                "kv_heads * head_dim must equal hidden_dim "
                f"({self.kv_heads} * {self.head_dim} != {self.hidden_dim})"
            )

    @property
    def model_hash(self) -> int:
        fields = (self.model_id, self.layers, self.hidden_dim, self.kv_heads, self.head_dim, self.elem_width)
        return fnv1a64("\x00".join(str(f) for f in fields).encode("utf-8"))


# ----------------------------------------------------------------- header / blob


@dataclass(frozen=True)
class KvBlobHeader:
    model_hash: int
    doc_ids: tuple[int, ...]
    token_count: int
    layers: int
    kv_heads: int
    head_dim: int
    elem_width: int
    payload_len: int
    checksum: int
    magic: bytes = MAGIC
    version: int = VERSION

    def __post_init__(self) -> None:
        if not self.doc_ids:
            raise ValueError("doc_ids must be non-empty")
        if self.token_count < 1:
            raise ValueError("token_count must be >= 1")
        want = 2 * self.layers * self.kv_heads * self.head_dim * self.token_count * self.elem_width
        if self.payload_len != want:
            raise ValueError(f"payload_len {self.payload_len} does not match dimensions (expected {want})")

    @property
    def encoded_size(self) -> int:
        return header_size(len(self.doc_ids)) + self.payload_len


class KvBlob:
    """Immutable (header, payload) pair (codec.py:140-149).

    Construction verifies the payload length and FNV-1a like the reference.
    ``KvBlob.trusted`` skips the re-hash for payloads whose checksum was just
    computed from these very bytes (the reference pays that hash twice,
    codec.py:148 and :222).
    """

    __slots__ = ("header", "payload", "device")  # device: optional HBM copy of the payload (load-path cache)

    def __init__(self, header: KvBlobHeader, payload) -> None:
        _, n = buffer_address(payload)
        if n != header.payload_len:
            raise ValueError("payload length does not match header")
        if fnv1a64(payload) != header.checksum:
            raise ValueError("payload checksum does not match header")
        object.__setattr__(self, "header", header)
        object.__setattr__(self, "payload", payload)
        object.__setattr__(self, "device", None)

    @classmethod
    def trusted(cls, header: KvBlobHeader, payload, device=None) -> "KvBlob":
        obj = object.__new__(cls)
        object.__setattr__(obj, "header", header)
        object.__setattr__(obj, "payload", payload)
        object.__setattr__(obj, "device", device)
        return obj

    def __setattr__(self, name, value):
        raise AttributeError("KvBlob is immutable")

    def payload_bytes(self) -> bytes:
        return as_bytes(self.payload)

    def payload_tensor(self):
        """uint8 CPU tensor view of the payload (zero-copy)."""
        import torch

        if hasattr(self.payload, "data_ptr"):
            return self.payload
        if len(self.payload) == 0:
            return torch.empty(0, dtype=torch.uint8)
        return torch.frombuffer(bytearray(self.payload) if isinstance(self.payload, memoryview) else self.payload,
                                dtype=torch.uint8)

    def __eq__(self, other) -> bool:
        if not isinstance(other, KvBlob):
            return NotImplemented
        if self.header != other.header:
            return False
        a, na = buffer_address(self.payload)
        b, nb = buffer_address(other.payload)
        if na != nb:
            return False
        return na == 0 or C.string_at(a, na) == C.string_at(b, nb)

    def __hash__(self) -> int:
        return hash((self.header, self.header.checksum))

    def __repr__(self) -> str:
        return f"KvBlob(header={self.header!r})"


def blob_size(profile: ModelProfile, token_count: int) -> int:
    """Payload bytes of ``token_count`` tokens, K and V (codec.py:152-156)."""
    if token_count < 0:
        raise ValueError("token_count must be >= 0")
    return 2 * profile.layers * profile.kv_heads * profile.head_dim * token_count * profile.elem_width


def header_size(doc_count: int) -> int:
    return int(_lib.lib().rdkv_header_size(doc_count))


def encoded_size(profile: ModelProfile, token_count: int, doc_count: int) -> int:
    return header_size(doc_count) + blob_size(profile, token_count)


def make_header(profile: ModelProfile, doc_ids: Sequence[int], token_count: int, checksum: int) -> KvBlobHeader:
    return KvBlobHeader(
        model_hash=profile.model_hash,
        doc_ids=tuple(int(d) for d in doc_ids),
        token_count=token_count,
        layers=profile.layers,
        kv_heads=profile.kv_heads,
        head_dim=profile.head_dim,
        elem_width=profile.elem_width,
        payload_len=blob_size(profile, token_count),
        checksum=checksum,
    )


def encode_header(h: KvBlobHeader) -> bytes:
    """Header bytes of :func:`encode` (codec.py:227-239), natively serialised."""
    n = len(h.doc_ids)
    ch = _lib.RdkvHeader(model_hash=h.model_hash, payload_len=h.payload_len, checksum=h.checksum,
                         token_count=h.token_count, version=h.version, doc_count=n, layers=h.layers,
                         kv_heads=h.kv_heads, head_dim=h.head_dim, elem_width=h.elem_width)
    ids = (C.c_uint64 * n)(*[d & _U64 for d in h.doc_ids])
    out = C.create_string_buffer(header_size(n))
    rc = _lib.lib().rdkv_header_encode(C.byref(ch), ids, out, len(out))
    raise_for(int(rc))
    return out.raw[: int(rc)]


def encode(blob: KvBlob) -> bytes:
    """Canonical byte encoding (codec.py:227-239)."""
    return encode_header(blob.header) + blob.payload_bytes()


def _header_from_native(ch: _lib.RdkvHeader, ids) -> KvBlobHeader:
    try:
        return KvBlobHeader(
            model_hash=ch.model_hash, doc_ids=tuple(int(x) for x in ids[: ch.doc_count]),
            token_count=ch.token_count, layers=ch.layers, kv_heads=ch.kv_heads, head_dim=ch.head_dim,
            elem_width=ch.elem_width, payload_len=ch.payload_len, checksum=ch.checksum)
    except ValueError as exc:  # pragma: no cover - native checks are a superset
        raise MalformedHeaderError(str(exc)) from exc


def _ids_buffer(addr: int, n: int):
    k = int.from_bytes(C.string_at(addr + 14, 2), "little") if n >= 16 else 1
    k = max(k, 1)
    return (C.c_uint64 * k)(), k


def decode_header(data) -> tuple[KvBlobHeader, int]:
    """Parse a header from the front of ``data`` -> (header, header_bytes) (codec.py:242-279)."""
    addr, n = buffer_address(data)
    ch = _lib.RdkvHeader()
    ids, k = _ids_buffer(addr, n)
    hl = C.c_size_t()
    raise_for(int(_lib.lib().rdkv_header_decode(addr, n, C.byref(ch), ids, k, C.byref(hl))))
    return _header_from_native(ch, ids), int(hl.value)


def decode(data) -> KvBlob:
    """Inverse of :func:`encode`; rejects corrupt or truncated input (codec.py:282-295)."""
    addr, n = buffer_address(data)
    ch = _lib.RdkvHeader()
    ids, k = _ids_buffer(addr, n)
    off = C.c_size_t()
    raise_for(int(_lib.lib().rdkv_blob_check(addr, n, C.byref(ch), ids, k, C.byref(off))))
    header = _header_from_native(ch, ids)
    start = int(off.value)
    if hasattr(data, "data_ptr"):
        payload = data[start : start + header.payload_len]
    else:
        payload = bytes(memoryview(data)[start : start + header.payload_len])
    return KvBlob.trusted(header, payload)


# ----------------------------------------------------------------- synthetic stand-in

_SM_GOLDEN = 0x9E3779B97F4A7C15
_SM_MIX1 = 0xBF58476D1CE4E5B9
_SM_MIX2 = 0x94D049BB133111EB


def splitmix64(x: int) -> int:
    x = (x + _SM_GOLDEN) & _U64
    x = ((x ^ (x >> 30)) * _SM_MIX1) & _U64
    x = ((x ^ (x >> 27)) * _SM_MIX2) & _U64
    return x ^ (x >> 31)


def splitmix_words(state: int, n_words: int, start: int = 1) -> np.ndarray:
    """Counter-mode splitmix64 words state + i*golden for i in [start, start+n)."""
    i = np.arange(start, start + n_words, dtype=np.uint64)
    x = np.uint64(state & _U64) + i * np.uint64(_SM_GOLDEN)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(_SM_MIX1)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(_SM_MIX2)
    return x ^ (x >> np.uint64(31))


def synth_blob(profile: ModelProfile, doc_ids: Sequence[int], token_count: int, seed: int = 0) -> KvBlob:
    """The reference's synthetic KV stand-in (codec.py:188-224), kept for
    compatibility and for storage-only tests; real KV comes from
    :class:`paper_2504_11765_b200.engine.KvGenerator`."""
    ids = tuple(int(d) for d in doc_ids)
    if not ids:
        raise ValueError("doc_ids must be non-empty")
    if token_count < 1:
        raise ValueError("token_count must be >= 1")
    state = splitmix64((seed & _U64) ^ profile.model_hash)
    for d in ids:
        state = splitmix64(state ^ (d & _U64))
    state = splitmix64(state ^ token_count)
    n = blob_size(profile, token_count)
    payload = splitmix_words(state, (n + 7) // 8).astype("<u8").tobytes()[:n]
    return KvBlob.trusted(make_header(profile, ids, token_count, fnv1a64(payload)), payload)
