"""Time rdkv_attention alone (CUDA events, warm) on a serving-shaped batch.

    python scripts/attn_perf.py [--seqs 32] [--new 64] [--cached 2560] [--dh 64] [--impl 0]
"""

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

from paper_2504_11765_b200 import _lib  # noqa: E402
from test_attention_gpu import _case, _ptr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=32)
    ap.add_argument("--new", type=int, default=64)
    ap.add_argument("--cached", type=int, default=2560)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--dh", type=int, default=64)
    ap.add_argument("--impl", type=int, default=0)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--same-block", action="store_true",
                    help="timing probe: every KV tile reads block 0 (L2-hot; outputs meaningless)")
    a = ap.parse_args()
    c = _case([a.new] * a.seqs, [a.cached] * a.seqs, a.hq, a.hkv, a.dh, shuffle=True)
    dev = "cuda"
    q, kp, vp = c["q"].to(dev), c["kp"].to(dev), c["vp"].to(dev)
    o = torch.empty_like(q)
    bt = c["bt"].to(dev)
    if a.same_block:
        bt.zero_()
    st, nn, nc = c["start"].to(dev), c["n_new"].to(dev), c["n_cached"].to(dev)
    lib = _lib.lib()
    nb = lib.rdkv_attention_scratch_bytes(c["T"], c["hq"], c["dh"])
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def call():
        _lib.check(lib.rdkv_attention(
            _ptr(q), a.hq * a.dh, _ptr(o), a.hq * a.dh, _ptr(kp), _ptr(vp), c["slots"], _ptr(st), _ptr(nn), _ptr(nc),
            _ptr(bt), bt.shape[1], 64, c["S"], c["T"], a.new, a.new + a.cached, a.hq, a.hkv, a.dh, a.impl, _ptr(ws),
            nb, C.c_void_p(stream.cuda_stream)))

    for _ in range(5):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    pairs = a.seqs * (a.new * a.cached + a.new * (a.new + 1) / 2)
    flops = 4.0 * a.dh * a.hq * pairs
    kv_bytes = a.seqs * (a.new + a.cached) * a.hkv * a.dh * 2 * 2
    print(json.dumps({"us": us, "tflops": flops / us / 1e6, "kv_gbs": kv_bytes / us / 1e3, "impl": a.impl,
                      "shape": vars(a)}))


if __name__ == "__main__":
    main()
