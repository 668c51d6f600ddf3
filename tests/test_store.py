"""KvStore parity: replay the reference's own op log (tests/golden/store_oplog.json,
produced by running ragdcache.store) and require identical outcomes, load costs,
counters, manifest bytes and recovery."""

import json
import os
import sys
import threading
from pathlib import Path

import pytest

from paper_2504_11765_b200 import codec
from paper_2504_11765_b200.codec import ModelProfile, synth_blob
from paper_2504_11765_b200.store import (CacheTier, CorruptBlobError, ImmutableEntryError, KeyMismatchError, KvKey,
                                         KvStore, Outcome, key_for, read_blob_file)

G = Path(__file__).resolve().parent / "golden"
LOG = json.loads((G / "store_oplog.json").read_text())
PROFILE = ModelProfile("tiny", 1, 4, 1, 4, 2)


def blob(ids, tokens=2, seed=0):
    return synth_blob(PROFILE, ids, tokens, seed=seed)


def test_replay_reference_oplog(tmp_path):
    st = KvStore(tmp_path / "s", memory_capacity_bytes=LOG["initial_capacity"])
    for op in LOG["ops"]:
        key = KvKey(PROFILE.model_hash, tuple(op["doc_ids"]))
        if op["op"] == "put":
            try:
                st.put(key, blob(op["doc_ids"], op["tokens"], op["seed"]))
                got = "ok"
            except ImmutableEntryError:
                got = "ImmutableEntryError"
            assert got == op["result"], op
        elif op["op"] == "get":
            r = st.get(key)
            assert r.outcome.value == op["result"], op
            assert r.load_cost_bytes == op["load_cost_bytes"], op
            assert (("%016x" % r.blob.header.checksum) if r.blob else None) == op["checksum"], op
        elif op["op"] == "contains":
            assert st.contains(key).value == op["result"], op
        else:
            st.set_memory_capacity(op["capacity"])
        assert json.loads(st.stats().to_json()) == op["stats"], op
    # manifest is byte-identical to the reference's
    assert (tmp_path / "s" / "manifest.jsonl").read_text().splitlines() == LOG["manifest"]
    re = KvStore(tmp_path / "s", memory_capacity_bytes=0)
    assert sorted(list(k.doc_ids) for k in re.keys()) == LOG["recovered_keys"]
    assert json.loads(re.stats().to_json()) == LOG["recovered_stats"]


def test_memory_vs_disk_hit(tmp_path):
    size = blob([1]).header.encoded_size
    st = KvStore(tmp_path, memory_capacity_bytes=10 * size)
    b = blob([1])
    st.put(key_for(PROFILE, [1]), b)
    r = st.get(key_for(PROFILE, [1]))
    assert r.outcome is Outcome.MEMORY_HIT and r.blob == b and r.load_cost_bytes == 0
    st2 = KvStore(tmp_path, memory_capacity_bytes=size - 1)
    st2.put(key_for(PROFILE, [1]), b)
    assert st2.contains(key_for(PROFILE, [1])) is CacheTier.ON_DISK
    r = st2.get(key_for(PROFILE, [1]))
    assert r.outcome is Outcome.DISK_HIT and r.blob == b and r.load_cost_bytes == size


@pytest.mark.parametrize("direct", ["0", "1"])
def test_disk_hit_payload_is_aligned_tensor(tmp_path, monkeypatch, direct):
    """Buffered reads put the payload on a 256-B boundary; O_DIRECT reads (the default)
    put the file's first byte on a 4096-B boundary.  Same bytes either way, for a blob
    smaller than one block and one that ends mid-block."""
    monkeypatch.setenv("RDKV_ODIRECT", direct)
    st = KvStore(tmp_path)
    for ids, tokens in (([5, 6], 3), ([7], 2900)):
        st.put(key_for(PROFILE, ids), blob(ids, tokens=tokens))
        r = KvStore(tmp_path).get(key_for(PROFILE, ids))
        assert r.outcome is Outcome.DISK_HIT
        hl = 46 + 8 * len(ids)
        if direct == "0":
            assert r.blob.payload.data_ptr() % 256 == 0
        else:
            assert (r.blob.payload.data_ptr() - hl) % 4096 == 0
        assert r.blob.payload_bytes() == blob(ids, tokens=tokens).payload


def test_immutability_and_noop_reput(tmp_path):
    st = KvStore(tmp_path)
    k = key_for(PROFILE, [1])
    st.put(k, blob([1]))
    m = (tmp_path / "manifest.jsonl").read_text()
    st.put(k, blob([1]))
    assert (tmp_path / "manifest.jsonl").read_text() == m
    with pytest.raises(ImmutableEntryError):
        st.put(k, blob([1], seed=1))
    with pytest.raises(KeyMismatchError):
        st.put(key_for(PROFILE, [2]), blob([1]))


def test_durability_bit_exact(tmp_path):
    st = KvStore(tmp_path)
    k, b = key_for(PROFILE, [5, 6]), blob([5, 6], tokens=3)
    st.put(k, b)
    path = tmp_path / f"{k.model_hash:016x}" / f"{k.file_stem}.rdkv"
    assert path.read_bytes() == codec.encode(b)


def test_corruption_quarantined(tmp_path):
    st = KvStore(tmp_path)
    k = key_for(PROFILE, [3])
    st.put(k, blob([3]))
    p = st.path_of(k)
    data = bytearray(p.read_bytes())
    data[-1] ^= 0xFF
    p.write_bytes(bytes(data))
    with pytest.raises(CorruptBlobError):
        st.get(k)
    assert not p.exists() and p.with_suffix(".rdkv.corrupt").exists()
    assert st.stats().corruptions == 1 and st.contains(k) is CacheTier.ABSENT
    assert st.get(k).outcome is Outcome.MISS


def test_torn_manifest_tail_tolerated(tmp_path):
    st = KvStore(tmp_path)
    st.put(key_for(PROFILE, [1]), blob([1]))
    with open(tmp_path / "manifest.jsonl", "a") as fh:
        fh.write('{"model_hash": "00')
    assert [k.doc_ids for k in KvStore(tmp_path).keys()] == [(1,)]


def test_concurrent_gets_and_puts(tmp_path):
    st = KvStore(tmp_path, memory_capacity_bytes=3 * blob([1]).header.encoded_size)
    errs = []

    def worker(seed):
        try:
            for i in range(60):
                ids = [1 + (i * 7 + seed) % 5]
                st.put(key_for(PROFILE, ids), blob(ids))
                assert st.get(key_for(PROFILE, ids)).outcome in (Outcome.MEMORY_HIT, Outcome.DISK_HIT)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(s,)) for s in range(8)]
    [t.start() for t in ths]
    [t.join() for t in ths]
    assert not errs
    s = st.stats()
    assert s.memory_bytes_used <= s.memory_capacity_bytes


@pytest.mark.skipif(not Path("/root/reference/pkg/src").exists(), reason="reference not mounted (GPU box)")
def test_reference_store_reads_our_files(tmp_path):
    """Files written by this store decode under, and are recovered by, the
    reference KvStore itself (checkpoint/resume cross-check)."""
    sys.path.insert(0, "/root/reference/pkg/src")
    from ragdcache import codec as rcodec, store as rstore
    st = KvStore(tmp_path)
    for ids in ([1], [4, 2], [9, 8, 7]):
        st.put(key_for(PROFILE, ids), blob(ids, tokens=len(ids)))
    ref = rstore.KvStore(tmp_path, memory_capacity_bytes=0)
    rp = rcodec.ModelProfile("tiny", 1, 4, 1, 4, 2)
    for ids in ([1], [4, 2], [9, 8, 7]):
        r = ref.get(rstore.key_for(rp, ids))
        assert r.outcome is rstore.Outcome.DISK_HIT
        assert r.blob.payload == blob(ids, tokens=len(ids)).payload


@pytest.mark.parametrize("direct", ["0", "1"])
def test_large_blob_file_roundtrip_parallel_read(tmp_path, monkeypatch, direct):
    monkeypatch.setenv("RDKV_ODIRECT", direct)
    # > 2 MiB files are read by several threads; sizes just past a piece boundary
    # must still include the tail bytes (header + payload + checksum verify)
    from paper_2504_11765_b200.codec import ModelProfile, synth_blob
    from paper_2504_11765_b200.store import KvKey, KvStore, Outcome
    prof = ModelProfile("tiny", 2, 256, 4, 64, 2)
    for tokens in (1025, 2049, 8192 + 3):             # 2 MiB + 2 KiB, 4 MiB + 2 KiB, 16 MiB + 6 KiB payloads
        key = KvKey(prof.model_hash, (tokens,))
        store = KvStore(tmp_path / str(tokens), memory_capacity_bytes=0)
        blob = synth_blob(prof, key.doc_ids, tokens)
        store.put(key, blob)
        look = store.get(key)
        assert look.outcome is Outcome.DISK_HIT
        assert look.blob == blob


@pytest.mark.parametrize("direct", [0, 1])
def test_file_read_range(tmp_path, direct):
    """rdkv_file_read_range (the streamed disk hit's segment reader): exact bytes for
    block-aligned ranges, short only at end of file, O_DIRECT alignment enforced."""
    import ctypes as C

    import numpy as np

    from paper_2504_11765_b200 import _lib

    data = np.random.default_rng(7).integers(0, 256, (5 << 20) + 1234, dtype=np.uint8)
    path = tmp_path / "f.bin"
    path.write_bytes(data.tobytes())
    L = _lib.lib()
    raw = np.zeros(len(data) + 3 * 4096, np.uint8)
    base = (-raw.ctypes.data) % 4096
    dst = raw.ctypes.data + base
    cap = len(raw) - base
    p = str(path).encode()
    for off, n in ((0, 4096), (4096, 3 << 20), (2 << 20, len(data) - (2 << 20)), (4 << 20, 8 << 20)):
        got = int(L.rdkv_file_read_range(p, C.c_void_p(dst), cap, off, n, direct))
        want = min(n, len(data) - off)
        assert got == want
        assert np.array_equal(raw[base: base + got], data[off: off + got])
    past = (len(data) + 4095) // 4096 * 4096 + 4096                                          # past the end
    assert int(L.rdkv_file_read_range(p, C.c_void_p(dst), cap, past, 4096, direct)) == 0
    if direct:
        assert int(L.rdkv_file_read_range(p, C.c_void_p(dst + 1), cap - 1, 0, 4096, 1)) < 0    # unaligned buffer
        assert int(L.rdkv_file_read_range(p, C.c_void_p(dst), cap, 100, 4096, 1)) < 0          # unaligned offset
