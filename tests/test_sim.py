"""Scheduler parity: the modeled executor reproduces the reference simulator
byte for byte (tests/golden/sim_small_report.json is the reference's own golden;
sim_runs.json holds more reference runs made by tests/golden/make_golden.py)."""

import json
from pathlib import Path

import pytest

from paper_2504_11765_b200.codec import ModelProfile
from paper_2504_11765_b200.costs import Configuration, CostParams, DeviceKind, DeviceProfile
from paper_2504_11765_b200.sim import (ArrivalProcess, ArrivalSpec, SimConfig, TopologyError, run,
                                       run_single_instance, service_capacity, sweep_rate)
from paper_2504_11765_b200.workload import zipf_stream

G = Path(__file__).resolve().parent / "golden"
MODEL = ModelProfile("sim-tiny", layers=2, hidden_dim=8, kv_heads=2, head_dim=4, elem_width=2)
PARAMS = CostParams(model=MODEL, network_delay=0.001)
RATE = 1.0e7


def gpu(name):
    return DeviceProfile(name, DeviceKind.INFERENCE_GPU, RATE)


DEVS = {
    "baseline": (gpu("gpu0"), gpu("gpu1")),
    "a": (gpu("gpu0"), DeviceProfile("gen0", DeviceKind.GENERATOR_GPU, RATE * 0.5)),
    "b": (gpu("gpu0"), gpu("gpu1"), DeviceProfile("cpu0", DeviceKind.CPU, RATE * 0.1)),
}


def test_reference_golden_snapshot_byte_for_byte():
    # reference test_sim.py:260-278
    cfg = SimConfig(configuration=Configuration.A, devices=DEVS["a"], cost=PARAMS,
                    arrival=ArrivalSpec(rate=100.0, process=ArrivalProcess.UNIFORM), k=2, tries=2, seed=1,
                    threshold=0.02, memory_capacity_bytes=0)
    report, records = run(cfg, zipf_stream(50, 1.0, 12, seed=3, k=2, q_tokens=16, doc_tokens=120))
    text = json.dumps({"report": report.to_dict(), "records": [r.to_dict() for r in records]}, sort_keys=True,
                      indent=1)
    assert text == (G / "sim_small_report.json").read_text()


RUNS = json.loads((G / "sim_runs.json").read_text())


@pytest.mark.parametrize("name", [n for n in RUNS if not n.startswith(("single", "sweep", "capacity"))])
def test_reference_runs(name):
    cfgname, proc, k, t, r, m = name.split("_")
    k, tries, rate, mem = int(k[1:]), int(t[1:]), float(r[1:]), int(m[1:])
    cfg = SimConfig(configuration=Configuration(cfgname), devices=DEVS[cfgname], cost=PARAMS,
                    arrival=ArrivalSpec(rate=rate, process=ArrivalProcess(proc)), k=k, tries=tries, seed=5,
                    threshold=0.03, memory_capacity_bytes=mem)
    report, records = run(cfg, zipf_stream(40, 1.0, 30, seed=2, k=k, q_tokens=16, doc_tokens=120))
    got = json.loads(json.dumps({"report": report.to_dict(), "records": [x.to_dict() for x in records]}))
    assert got == RUNS[name]


@pytest.mark.parametrize("b,use", [(1, True), (1, False), (4, True), (4, False)])
def test_single_instance(b, use):
    cfg = SimConfig(configuration=Configuration.SINGLE_INSTANCE, devices=(gpu("gpu0"),), cost=PARAMS,
                    arrival=ArrivalSpec(rate=10.0), k=1, tries=1, seed=1, threshold=0.5, memory_capacity_bytes=2000)
    rep, recs = run_single_instance(cfg, zipf_stream(40, 1.0, 25, seed=4, k=2, q_tokens=16, doc_tokens=120),
                                    batch_size=b, use_cache=use)
    got = json.loads(json.dumps({"report": rep.to_dict(), "records": [r.to_dict() for r in recs]}))
    assert got == RUNS[f"single_b{b}_{use}"]


def test_sweep_and_capacity():
    cfg = SimConfig(configuration=Configuration.BASELINE, devices=DEVS["baseline"], cost=PARAMS,
                    arrival=ArrivalSpec(rate=50.0), k=1, tries=1, seed=1, threshold=0.05)
    items = zipf_stream(50, 1.0, 20, seed=1, k=1, q_tokens=16, doc_tokens=120)
    assert [p.to_dict() for p in sweep_rate(cfg, [5.0, 20.0, 80.0], items)] == RUNS["sweep"]
    assert service_capacity(cfg, items) == RUNS["capacity"]


def test_topology_validation():
    with pytest.raises(TopologyError):
        SimConfig(configuration=Configuration.A, devices=DEVS["baseline"], cost=PARAMS, arrival=ArrivalSpec(1.0))
    with pytest.raises(TopologyError):
        SimConfig(configuration=Configuration.BASELINE, devices=DEVS["a"], cost=PARAMS, arrival=ArrivalSpec(1.0))
    cfg = SimConfig(configuration=Configuration.SHARED_GPU_N, devices=tuple(gpu(f"gpu{i}") for i in range(8)),
                    cost=PARAMS, arrival=ArrivalSpec(1.0))
    assert len(cfg.instances) == 8 and not cfg.prefetch_enabled


def test_invariants_n_instances():
    devs = tuple(gpu(f"gpu{i}") for i in range(4)) + (DeviceProfile("gen", DeviceKind.GENERATOR_GPU, RATE),)
    cfg = SimConfig(configuration=Configuration.SHARED_GPU_N, devices=devs, cost=PARAMS, arrival=ArrivalSpec(400.0),
                    k=3, tries=3, seed=2, threshold=0.01)
    report, recs = run(cfg, zipf_stream(30, 1.0, 60, seed=9, k=3, q_tokens=16, doc_tokens=120))
    assert report.completed == 180
    for r in recs:  # TTFT decomposition (reference test_sim.py:121-165)
        assert abs(r.queue_wait + r.kv_load + r.prefill + r.network_delay - (r.first_token - r.arrival)) <= 1e-9
    by_inst = {}
    for r in recs:
        by_inst.setdefault((r.try_index, r.instance_id), []).append(r)
    for rows in by_inst.values():  # an instance serves one query at a time
        rows.sort(key=lambda r: r.dispatch)
        for a, b in zip(rows, rows[1:]):
            assert b.dispatch >= a.dispatch + a.kv_load + a.prefill - 1e-12
    assert report.origin_counts.get("generated", 0) > 0


def test_calibrated_executor_uses_measured_costs():
    """serving.CalibratedExecutor answers the policy from a B200 cost table:
    prefill by cached-prefix level, per-byte load by tier, generation by length."""
    from paper_2504_11765_b200.costs import (Configuration, CostParams, DeviceKind, DeviceProfile, ModelProfile,
                                             Tier)
    from paper_2504_11765_b200.serving import CalibratedExecutor
    from paper_2504_11765_b200.sim import ArrivalSpec, Dispatch, GenTask, SimConfig, run
    from paper_2504_11765_b200.workload import zipf_stream

    costs = {"k": 2, "prefill_s_by_cached_docs": [0.03, 0.02, 0.01], "host_tier_load_s_per_byte": 1e-11,
             "disk_read_verify_s_per_byte": 1e-9, "generation_s_by_docs": [0.05, 0.09]}
    prof = ModelProfile("m", 2, 8, 2, 4, 2)
    devs = tuple(DeviceProfile(f"g{i}", DeviceKind.INFERENCE_GPU, 1.0) for i in range(2))
    cfg = SimConfig(configuration=Configuration.SHARED_GPU_N, devices=devs, cost=CostParams(model=prof),
                    arrival=ArrivalSpec(rate=5.0), k=2, tries=1, seed=3)
    ex = CalibratedExecutor(costs)
    ex.bind(cfg, None)
    it = zipf_stream(50, 1.0, 1, seed=0, k=2, q_tokens=4, doc_tokens=8)[0]
    miss = Dispatch(0, it, it.doc_ids[:2], it.doc_tokens[:2], 0, None, 0, 20, 0)
    assert ex.serve(miss) == (0.0, 0.03)
    disk = Dispatch(0, it, it.doc_ids[:2], it.doc_tokens[:2], 1, Tier.DISK, 8, 12, 1000)
    assert ex.serve(disk) == (1000 * 1e-9, 0.02)
    mem = Dispatch(0, it, it.doc_ids[:2], it.doc_tokens[:2], 2, Tier.MEMORY, 16, 4, 1000)
    assert ex.serve(mem) == (1000 * 1e-11, 0.01)
    peer = CalibratedExecutor(costs, memory_tier_s_per_byte=2e-12)  # C4 "P2P on": memory tier = pooled peer HBM
    peer.bind(cfg, None)
    assert peer.serve(mem) == (1000 * 2e-12, 0.01) and peer.serve(disk) == (1000 * 1e-9, 0.02)
    assert ex.generation_time(GenTask(it.doc_ids[:2], 16, 100)) == 0.09
    report, records = run(cfg, zipf_stream(50, 1.0, 20, seed=0, k=2, q_tokens=4, doc_tokens=8), CalibratedExecutor(costs))
    assert len(records) == 20 and all(r.prefill == 0.03 for r in records)   # no generator: every query misses
