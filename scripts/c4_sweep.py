"""C4 projection: the reference scheduling policy (sim.run) with 8
Llama-3-8B-shaped serving instances, queue-time proactive precompute on a
generator, Zipf(1.0) over 10k docs, k=10 x 512 + 64, Poisson arrivals swept
toward saturation — every cost a B200 measurement from one GPU
(profiles/r1_b200_costs_8b.json via serving.CalibratedExecutor).  Modeled,
not measured on 8 GPUs: the driver's SCALE run measures the replicas.

    python scripts/c4_sweep.py > profiles/r1_c4_projection.jsonl
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_11765_b200.costs import Configuration, CostParams, DeviceKind, DeviceProfile
from paper_2504_11765_b200.model import get_spec
from paper_2504_11765_b200.serving import CalibratedExecutor, summarize
from paper_2504_11765_b200.sim import ArrivalSpec, SimConfig, run
from paper_2504_11765_b200.workload import zipf_stream

ROOT = Path(__file__).resolve().parents[1]
costs = json.loads((ROOT / "profiles" / "r1_b200_costs_8b.json").read_text())
spec = get_spec("llama-3-8b")
items = zipf_stream(10000, 1.0, 2000, seed=1, k=10, q_tokens=64, doc_tokens=512)
full = costs["prefill_s_by_cached_docs"][0]
cap = 8 / full  # all-miss capacity of 8 instances
# "P2P on": the memory tier is the 8 instances' pooled HBM KV tiers (100 GiB each),
# a hit fetched from the holder over NVLink by the K3p gather (modeled: NVLink 5 at
# 0.85 x 900 GB/s; one GPU here cannot measure it).  "P2P off": the shared pinned
# host tier (256 GiB) at the measured layer-streamed H2D cost.
NVLINK_S_PER_BYTE = 1.0 / (0.85 * 900e9)
configs = ((False, 0, None, "none"), (True, 0, None, "none"), (True, 256 << 30, None, "host tier (P2P off)"),
           (True, 8 * (100 << 30), NVLINK_S_PER_BYTE, "peer HBM tier (P2P on, modeled NVLink)"))
for gen, mem, mem_cost, tier in configs:
    for frac in (0.5, 1.0, 1.5, 2.0, 3.0):
        rate = cap * frac
        devs = tuple(DeviceProfile(f"b200-{i}", DeviceKind.INFERENCE_GPU, 1.0) for i in range(8))
        if gen:
            devs += (DeviceProfile("b200-gen", DeviceKind.GENERATOR_GPU, 1.0),)
        cfg = SimConfig(configuration=Configuration.SHARED_GPU_N, devices=devs,
                        cost=CostParams(model=spec.profile(), network_delay=0.0), arrival=ArrivalSpec(rate=rate),
                        k=10, tries=3, seed=1, threshold=0.5, memory_capacity_bytes=mem)
        report, records = run(cfg, items, CalibratedExecutor(costs, memory_tier_s_per_byte=mem_cost))
        s = summarize(records)
        tries = report.per_try
        print(json.dumps({"instances": 8, "generator": gen, "memory_tier": tier, "memory_tier_bytes": mem,
                          "rate_qps": rate,
                          "rate_over_all_miss_capacity": frac,
                          "qps_per_try": [t.throughput for t in tries],
                          "latency_median_ms_per_try": [t.latency_median * 1e3 for t in tries],
                          "latency_p95_ms_per_try": [t.latency_p95 * 1e3 for t in tries],
                          "ttft_ms": s["ttft_ms"], "origins": s["origins"]}), flush=True)
