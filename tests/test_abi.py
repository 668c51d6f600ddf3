"""librdkv loads and exports every symbol include/rdkv.h declares (no GPU needed)."""

import re
from pathlib import Path

from paper_2504_11765_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "rdkv.h"


def declared_symbols():
    return re.findall(r"RDKV_API\s+[\w\s\*]+?\b(rdkv_\w+)\s*\(", HEADER.read_text())


def test_header_declares_the_path():
    names = set(declared_symbols())
    for must in ("rdkv_fnv1a64", "rdkv_blob_read", "rdkv_blob_write", "rdkv_kv_unpack", "rdkv_model_create",
                 "rdkv_forward", "rdkv_gemm_bf16"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version():
    assert _lib.lib().rdkv_abi_version() == 1


def test_python_signatures_cover_host_symbols():
    # every host-side entry point has a ctypes signature in _lib.SIGNATURES
    host = {n for n in declared_symbols() if not n.startswith(("rdkv_model", "rdkv_forward", "rdkv_workspace",
                                                               "rdkv_kv_unpack", "rdkv_kv_stream", "rdkv_kv_copy", "rdkv_kv_peer", "rdkv_ipc", "rdkv_tp", "rdkv_memcpy", "rdkv_profile"))}
    assert host <= set(_lib.SIGNATURES), host - set(_lib.SIGNATURES)
