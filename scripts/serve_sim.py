"""Reference scheduling policy (sim.run) driven by measured B200 execution.

Config A of the paper on B200 timing: one serving instance + one queue-time
generator, Poisson arrivals, Zipf(1.0) doc locality, `tries` passes with the
cache persisting (sim.py:343-355).  Prints a JSON summary; with --compare also
runs the BASELINE topology (no generator) on the same workload.

  python scripts/serve_sim.py --model llama-3.2-1b --k 5 --queries 120 --rate 200
"""
import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2504_11765_b200.costs import Configuration, CostParams, DeviceKind, DeviceProfile
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.model import get_spec
from paper_2504_11765_b200.service import SharedCacheService
from paper_2504_11765_b200.serving import MeasuredExecutor, summarize
from paper_2504_11765_b200.sim import ArrivalSpec, SimConfig, run
from paper_2504_11765_b200.store import GpuVerifier, KvStore
from paper_2504_11765_b200.workload import zipf_stream


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-3.2-1b")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--doc-tokens", type=int, default=512)
    ap.add_argument("--q-tokens", type=int, default=64)
    ap.add_argument("--queries", type=int, default=120)
    ap.add_argument("--docs", type=int, default=10000)
    ap.add_argument("--rate", type=float, default=200.0)
    ap.add_argument("--tries", type=int, default=2)
    ap.add_argument("--threshold", type=float, default=0.005)
    ap.add_argument("--configuration", default="a", choices=["a", "baseline_1"])
    a = ap.parse_args()

    spec = get_spec(a.model, a.layers)
    eng = Engine(spec, seed=0, pool_tokens=a.k * a.doc_tokens + a.q_tokens + 4096)
    root = Path(tempfile.mkdtemp(prefix="rdkv_serve_"))
    svc = SharedCacheService(KvStore(root, memory_capacity_bytes=0, verifier=GpuVerifier(eng.device)))
    inst = DeviceProfile("b200-0", DeviceKind.INFERENCE_GPU, 1.0)
    if a.configuration == "a":
        cfg_kind, devices = Configuration.SHARED_GPU_N, (inst, DeviceProfile("b200-gen", DeviceKind.GENERATOR_GPU, 1.0))
    else:
        cfg_kind, devices = Configuration.SHARED_GPU_N, (inst,)
    cfg = SimConfig(configuration=cfg_kind, devices=devices, cost=CostParams(model=spec.profile(), network_delay=0.0),
                    arrival=ArrivalSpec(rate=a.rate), k=a.k, tries=a.tries, seed=1, threshold=a.threshold,
                    memory_capacity_bytes=0)
    items = zipf_stream(a.docs, 1.0, a.queries, seed=1, k=a.k, q_tokens=a.q_tokens, doc_tokens=a.doc_tokens)
    ex = MeasuredExecutor(eng, svc, workload={it.query_id: it for it in items})
    t0 = time.perf_counter()
    report, records = run(cfg, items, ex)
    wall = time.perf_counter() - t0
    out = {"model": spec.name, "layers": spec.layers, "k": a.k, "rate": a.rate, "tries": a.tries,
           "configuration": a.configuration, "wall_s": wall, "summary": summarize(records, ex.access_log),
           "per_try": [{"try": t.try_index, "qps": t.throughput, "latency_median_ms": t.latency_median * 1e3,
                        "latency_p95_ms": t.latency_p95 * 1e3, "disk_hit_ratio": t.disk_hit_ratio,
                        "miss_ratio": t.miss_ratio} for t in report.per_try],
           "generations": len(ex.generations),
           "gen_ms_mean": 1e3 * sum(g for _, g in ex.generations) / max(1, len(ex.generations)),
           "mirror_vs_store": sum(1 for x in ex.access_log if (x.mirror_tier == "miss") != (x.outcome == "miss"))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
