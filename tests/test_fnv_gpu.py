"""Parallel FNV-1a on the GPU (rdkv_fnv1a64_device) is bit-exact with the
serial definition (codec.py:64-69): the reference's own vectors
(tests/golden/codec_golden.json, produced by the reference), the C oracle on
random buffers at chunk-boundary lengths and seeds, and the disk-hit path of
the store with the GPU verifier (good file -> DISK_HIT with the HBM copy
attached; flipped payload byte -> CorruptBlobError + quarantine, like the host
check)."""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle.codec_ref import fnv1a64 as oracle_fnv
from paper_2504_11765_b200 import codec
from paper_2504_11765_b200.codec import FNV_OFFSET, ModelProfile, fnv1a64_device, synth_blob
from paper_2504_11765_b200.store import CorruptBlobError, GpuVerifier, KvKey, KvStore, Outcome

pytestmark = pytest.mark.gpu
GOLDEN = json.loads((Path(__file__).parent / "golden" / "codec_golden.json").read_text())


def _dev(b: bytes) -> torch.Tensor:
    return torch.tensor(list(b), dtype=torch.uint8, device="cuda") if b else torch.empty(0, dtype=torch.uint8,
                                                                                         device="cuda")


def test_reference_vectors():
    for v in GOLDEN["fnv"]:
        assert fnv1a64_device(_dev(bytes.fromhex(v["hex"]))) == int(v["hash"], 16)
    for v in GOLDEN["fnv_seeded"]:
        assert fnv1a64_device(_dev(bytes.fromhex(v["hex"])), int(v["seed"], 16)) == int(v["hash"], 16)


@pytest.mark.parametrize("n", [1, 3, 15, 16, 17, 4095, 4096, 4097, 16383, 16384, 16385, 65536 * 3 + 7, 1 << 20])
def test_random_buffers_match_serial(n):
    rng = np.random.default_rng(n)
    host = rng.integers(0, 256, n, dtype=np.uint8)
    dev = torch.from_numpy(host).cuda()
    for seed in (FNV_OFFSET, 0, 0x0123456789ABCDEF):
        assert fnv1a64_device(dev, seed) == oracle_fnv(host.tobytes(), seed)
    # an unaligned view (exercises the byte-load paths)
    assert fnv1a64_device(dev[1:]) == oracle_fnv(host[1:].tobytes(), FNV_OFFSET)


@pytest.mark.parametrize("n", [1, 16384, 16385, 5 * 16384 + 77, 1 << 20])
def test_streaming_fnv_matches_one_shot(n):
    """codec.StreamingFnv (the automaton pass per landed segment, then the rest) gives the
    one-shot checksum whatever the segment boundaries (mid-chunk, repeated, past the end)."""
    rng = np.random.default_rng(n + 1)
    host = rng.integers(0, 256, n, dtype=np.uint8)
    dev = torch.from_numpy(host).cuda()
    want = oracle_fnv(host.tobytes(), FNV_OFFSET)
    for steps in ([], [n // 3, n // 3, 2 * n // 3 + 1], [16383, 16384, 40000, n + 5]):
        s = codec.StreamingFnv(dev)
        for r in steps:
            s.advance(r)
        assert s.result() == want, (n, steps)


def test_large_payload_matches_native():
    x = torch.randint(0, 256, (80 << 20,), dtype=torch.uint8, device="cuda")   # one C2 composite
    assert fnv1a64_device(x) == codec.fnv1a64(x.cpu())


def test_store_gpu_verified_disk_hit_and_corruption(tmp_path):
    prof = ModelProfile("tiny", 2, 256, 4, 64, 2)
    key = KvKey(prof.model_hash, (3, 8))
    blob = synth_blob(prof, key.doc_ids, 40)
    store = KvStore(tmp_path, memory_capacity_bytes=0, verifier=GpuVerifier("cuda"))
    store.put(key, blob)
    look = store.get(key)
    assert look.outcome is Outcome.DISK_HIT
    assert look.blob.device is not None and look.blob.device.is_cuda
    assert torch.equal(look.blob.device.cpu(), look.blob.payload_tensor())
    # corrupt one payload byte on disk: same outcome class as the host verifier
    path = store.path_of(key)
    raw = bytearray(path.read_bytes())
    raw[-5] ^= 0x40
    path.write_bytes(bytes(raw))
    with pytest.raises(CorruptBlobError):
        store.get(key)
    assert store.contains(key).name == "ABSENT"
