"""Streamed disk hits (store._read_streamed): a blob file larger than one 64-MiB read
segment is read segment by segment, each segment's payload copied to HBM while the next
is read, and checksummed on the GPU.  Same bytes, same tiers and the same exceptions
(checksum mismatch -> CorruptBlobError + quarantine, truncation) as the one-shot read."""

import pytest
import torch

from paper_2504_11765_b200 import _lib, store as store_mod
from paper_2504_11765_b200.codec import ModelProfile, synth_blob
from paper_2504_11765_b200.store import CorruptBlobError, GpuVerifier, KvKey, KvStore, Outcome

pytestmark = pytest.mark.gpu

PROF = ModelProfile("tiny", 2, 256, 4, 64, 2)   # 2 KiB of payload per token


@pytest.fixture(scope="module")
def big():
    tokens = 36_000 + 7                             # ~70 MiB: two segments, ragged tail
    key = KvKey(PROF.model_hash, (tokens,))
    return key, synth_blob(PROF, key.doc_ids, tokens)


@pytest.mark.parametrize("direct", ["1", "0"])
def test_streamed_disk_hit_matches(tmp_path, monkeypatch, big, direct):
    monkeypatch.setenv("RDKV_ODIRECT", direct)
    key, blob = big
    KvStore(tmp_path, memory_capacity_bytes=0).put(key, blob)
    st = KvStore(tmp_path, memory_capacity_bytes=0, verifier=GpuVerifier("cuda"))
    assert st.path_of(key).stat().st_size > store_mod._STREAM_SEG
    _lib.lib().rdkv_drop_page_cache(str(st.path_of(key)).encode())
    look = st.get(key)
    assert look.outcome is Outcome.DISK_HIT
    assert look.blob.header == blob.header
    want = blob.payload_tensor()
    assert torch.equal(look.blob.payload_tensor(), want)
    assert look.blob.device is not None and torch.equal(look.blob.device.cpu(), want)


def test_streamed_checksum_mismatch_quarantines(tmp_path, big):
    key, blob = big
    st = KvStore(tmp_path, memory_capacity_bytes=0, verifier=GpuVerifier("cuda"))
    st.put(key, blob)
    p = st.path_of(key)
    with open(p, "r+b") as fh:                      # flip a byte in the second segment
        fh.seek(store_mod._STREAM_SEG + 12345)
        b = fh.read(1)
        fh.seek(store_mod._STREAM_SEG + 12345)
        fh.write(bytes([b[0] ^ 0x5A]))
    with pytest.raises(CorruptBlobError):
        st.get(key)
    assert not p.exists() and p.with_suffix(".rdkv.corrupt").exists()


def test_streamed_truncated_file_is_corrupt(tmp_path, big):
    key, blob = big
    st = KvStore(tmp_path, memory_capacity_bytes=0, verifier=GpuVerifier("cuda"))
    st.put(key, blob)
    p = st.path_of(key)
    with open(p, "r+b") as fh:
        fh.truncate(p.stat().st_size - 4096 - 3)
    with pytest.raises(CorruptBlobError):
        st.get(key)
