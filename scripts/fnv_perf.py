"""FNV-1a of one cached-KV payload: GPU (parallel, bit-exact) vs one host core."""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_11765_b200 import codec

out = []
for mib in (16, 80, 640):   # C2 doc, C2 composite, C3 composite
    x = torch.randint(0, 256, (mib << 20,), dtype=torch.uint8, device="cuda")
    h = x.cpu().pin_memory()
    codec.fnv1a64_device(x)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        a = codec.fnv1a64_device(x)
    gpu = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    b = codec.fnv1a64(h)
    cpu = time.perf_counter() - t0
    assert a == b
    out.append({"MiB": mib, "gpu_ms": gpu * 1e3, "gpu_GBps": (mib << 20) / gpu / 1e9, "host_core_ms": cpu * 1e3,
                "host_GBps": (mib << 20) / cpu / 1e9, "speedup": cpu / gpu})
print(json.dumps(out))
