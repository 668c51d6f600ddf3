"""The reference scheduling policy driven by measured B200 execution (SURVEY H-i):
every dispatch does the real lookup/load/prefill, every generation the real
document prefill + put; the store's real outcomes agree with the policy mirror."""

import pytest

from paper_2504_11765_b200.costs import Configuration, CostParams, DeviceKind, DeviceProfile
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.model import get_spec
from paper_2504_11765_b200.service import SharedCacheService
from paper_2504_11765_b200.serving import MeasuredExecutor, summarize
from paper_2504_11765_b200.sim import ArrivalSpec, SimConfig, run
from paper_2504_11765_b200.store import KvKey, KvStore
from paper_2504_11765_b200.workload import zipf_stream

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cap", [0, 600_000])
def test_measured_policy_run(tmp_path, cap):
    spec = get_spec("gqa-small-64")
    eng = Engine(spec, seed=2, pool_tokens=8192)
    store = KvStore(tmp_path, memory_capacity_bytes=cap)
    store.oplog = []
    svc = SharedCacheService(store)
    devs = (DeviceProfile("gpu0", DeviceKind.INFERENCE_GPU, 1.0), DeviceProfile("gen", DeviceKind.GENERATOR_GPU, 1.0))
    cfg = SimConfig(configuration=Configuration.SHARED_GPU_N, devices=devs,
                    cost=CostParams(model=spec.profile(), network_delay=0.0), arrival=ArrivalSpec(rate=1.0e6),
                    k=3, tries=2, seed=1, threshold=0.0, memory_capacity_bytes=cap)
    items = zipf_stream(30, 1.0, 40, seed=3, k=3, q_tokens=16, doc_tokens=64)
    ex = MeasuredExecutor(eng, svc)
    report, records = run(cfg, items, ex)
    assert report.completed == 80 and len(ex.access_log) == 80
    # the real store agrees with the policy's mirror on every decision
    for a in ex.access_log:
        assert (a.mirror_tier == "miss") == (a.outcome == "miss")
        if cap == 0:
            assert a.mirror_tier != "memory"  # capacity 0: the memory tier is off (paper.json)
    # every generated prefix is durable in the store
    for ids, _ in ex.generations:
        assert svc.contains(KvKey(spec.profile().model_hash, ids)).value in ("on_disk", "in_memory")
    assert ex.generations and any(a.outcome == "disk_hit" for a in ex.access_log)
    for r in records:
        assert abs(r.queue_wait + r.kv_load + r.prefill - (r.first_token - r.arrival)) < 1e-9
    s = summarize(records, ex.access_log)
    assert s["qps"] > 0 and s["ttft_ms"]["p99"] >= s["ttft_ms"]["p50"]
    # SURVEY H-i: the real store's operation log replays into the reference store law
    from dataclasses import asdict

    from oracle.store_ref import replay_oplog as replay

    want = replay(store.oplog, cap)
    got = asdict(store.stats())
    assert all(got[f] == v for f, v in want.items()), (got, want)
    if cap:
        assert any(a.outcome == "memory_hit" for a in ex.access_log)
