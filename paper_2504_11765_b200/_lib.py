"""ctypes binding of librdkv.so (include/rdkv.h).

ctypes releases the GIL for the duration of every foreign call, so the worker
threads of the scheduler run GPU launches and blob I/O concurrently.  There is
no fallback: if the library is missing every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import os

# RDKV_LIB points at an alternative build (A/B measurements of kernel variants)
LIB_PATH = Path(os.environ.get("RDKV_LIB") or Path(__file__).resolve().parent / "librdkv.so")

RDKV_OK = 0
RDKV_ERR_BAD_MAGIC = -1
RDKV_ERR_UNSUPPORTED_VERSION = -2
RDKV_ERR_TRUNCATED = -3
RDKV_ERR_CHECKSUM = -4
RDKV_ERR_MALFORMED = -5
RDKV_ERR_IO = -6
RDKV_ERR_ARG = -7
RDKV_ERR_CUDA = -8

EPI_STORE = 0
EPI_STORE_F32 = 1
EPI_RESID = 2
EPI_SWIGLU = 3


class RdkvHeader(C.Structure):
    _fields_ = [
        ("model_hash", C.c_uint64),
        ("payload_len", C.c_uint64),
        ("checksum", C.c_uint64),
        ("token_count", C.c_uint32),
        ("version", C.c_uint16),
        ("doc_count", C.c_uint16),
        ("layers", C.c_uint16),
        ("kv_heads", C.c_uint16),
        ("head_dim", C.c_uint16),
        ("elem_width", C.c_uint8),
        ("reserved_pad", C.c_uint8 * 3),
    ]


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str) -> None:
        super().__init__(f"librdkv error {code}: {message}")
        self.code = code


_u64, _i64, _sz, _vp, _cp, _i32 = C.c_uint64, C.c_int64, C.c_size_t, C.c_void_p, C.c_char_p, C.c_int

# symbol -> (restype, argtypes); mirrors include/rdkv.h
SIGNATURES: dict[str, tuple] = {
    "rdkv_abi_version": (_i32, []),
    "rdkv_last_error": (_cp, []),
    "rdkv_fnv1a64": (_u64, [_vp, _sz, _u64]),
    "rdkv_fnv1a64_many": (None, [C.POINTER(_vp), C.POINTER(_sz), _sz, C.POINTER(_u64), _i32]),
    "rdkv_header_size": (_sz, [C.c_uint32]),
    "rdkv_header_encode": (_i64, [C.POINTER(RdkvHeader), C.POINTER(_u64), _vp, _sz]),
    "rdkv_header_decode": (_i32, [_vp, _sz, C.POINTER(RdkvHeader), C.POINTER(_u64), _sz, C.POINTER(_sz)]),
    "rdkv_blob_check": (_i32, [_vp, _sz, C.POINTER(RdkvHeader), C.POINTER(_u64), _sz, C.POINTER(_sz)]),
    "rdkv_blob_write": (_i32, [_cp, _cp, _vp, _sz, _vp, _sz]),
    "rdkv_file_size": (_i64, [_cp]),
    "rdkv_blob_read": (_i32, [_cp, _vp, _sz, _sz, _i32, C.POINTER(RdkvHeader), C.POINTER(_u64), _sz,
                              C.POINTER(_sz), C.POINTER(_sz)]),
    "rdkv_file_read_range": (_i64, [_cp, _vp, _sz, _u64, _sz, _i32]),
    "rdkv_drop_page_cache": (_i32, [_cp]),
    "rdkv_gemm_bf16": (_i32, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _vp]),
    "rdkv_fnv1a64_device_scratch": (_sz, [_sz]),
    "rdkv_fnv1a64_device": (_i32, [_vp, _sz, _u64, _vp, _sz, _vp, _vp]),
    "rdkv_fnv1a64_device_partial": (_i64, [_vp, _sz, _sz, _i64, _vp, _sz, _vp]),
    "rdkv_fnv1a64_device_finish": (_i32, [_vp, _sz, _u64, _vp, _sz, _vp, _vp]),
    "rdkv_attention": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32,
                              _i32, _i32, _i32, _i32, _i32, _vp, _sz, _vp]),
    "rdkv_attention_scratch_bytes": (_sz, [_i32, _i32, _i32]),
    "rdkv_gemm_bf16_ex": (_i32, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _sz,
                                 _vp]),
    # node control plane (csrc/shm.cpp)
    "rdkv_shm_open": (_i32, [_cp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, C.POINTER(_vp)]),
    "rdkv_shm_close": (None, [_vp]),
    "rdkv_shm_unlink": (_i32, [_cp]),
    "rdkv_shm_world": (_i32, [_vp]),
    "rdkv_shm_key_state": (_i32, [_vp, _u64, _u64, C.POINTER(_i32)]),
    "rdkv_shm_key_cas": (_i32, [_vp, _u64, _u64, _i32, _i32, _i32]),
    "rdkv_shm_res_publish": (_i32, [_vp, _u64, _u64, _i32, C.POINTER(C.c_int32), _i32, _i32]),
    "rdkv_shm_res_pin": (_i32, [_vp, _u64, _u64, C.POINTER(_i32), C.POINTER(C.c_int32), _i32, C.POINTER(_i32)]),
    "rdkv_shm_res_unpin": (_i32, [_vp, _u64, _u64]),
    "rdkv_shm_res_retract": (_i32, [_vp, _u64, _u64, _i32]),
    "rdkv_shm_res_holder": (_i32, [_vp, _u64, _u64]),
    "rdkv_shm_ring_push": (_i32, [_vp, _i32, _vp, _i32]),
    "rdkv_shm_ring_pop": (_i32, [_vp, _i32, _vp, _i32]),
    "rdkv_shm_ring_size": (_i64, [_vp, _i32]),
    "rdkv_shm_qstate_cas": (_i32, [_vp, _i32, _i32, _i32]),
    "rdkv_shm_qstate": (_i32, [_vp, _i32]),
    "rdkv_shm_counter_add": (_i64, [_vp, _i32, _i64]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load librdkv.so once (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing; build it with `python -m paper_2504_11765_b200.build` "
                    "(there is no CPU fallback)"
                )
            handle = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error() -> str:
    return (lib().rdkv_last_error() or b"").decode("utf-8", "replace")


def check(rc: int) -> int:
    """Raise NativeError for a negative status code."""
    if rc < 0:
        raise NativeError(int(rc), last_error())
    return rc
