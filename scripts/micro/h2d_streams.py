"""Pinned host -> HBM copy bandwidth with 1, 2 and 4 concurrent streams (copy engines)."""
import json
import torch

n = 1 << 30
src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
out = {}
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = n // k
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        out[f"streams_{k}"] = n / (e0.elapsed_time(e1) / 1e3) / 1e9
print(json.dumps(out))
