"""K1 at the C3 bench shapes (M = 16 queries x 64 tokens = 1024 rows, Llama-3-8B
projections): every tile plan vs cuBLAS (torch.matmul, no epilogue), and a K sweep
of the planner's choice to separate the fixed cost from the per-k-block cost.

    python scripts/gemm_c3.py > profiles/r2_gemm_c3.txt
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2504_11765_b200 import _lib


FLUSH = None


def t_gemm(M, N, K, epi, tile, iters=30, cold=False):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    n_out = N // 2 if epi == _lib.EPI_SWIGLU else N
    D = torch.empty(M, n_out, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    L = _lib.lib()
    f = lambda: _lib.check(L.rdkv_gemm_bf16_ex(A.data_ptr(), K, B.data_ptr(), K, D.data_ptr(), n_out, None, 0, M, N,
                                               K, epi, tile, None, 0, s))
    try:
        for _ in range(3):
            f()
    except Exception:
        return float("nan")
    if cold:  # weights and activations evicted from L2 before every launch (as inside the step)
        global FLUSH
        if FLUSH is None:
            FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        evs = []
        for _ in range(iters):
            FLUSH.fill_(1)  # ~80 us of device work: the launch below is enqueued before it ends
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs) / iters * 1e3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def t_cublas(M, N, K, iters=30):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        torch.matmul(A, B.T)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        torch.matmul(A, B.T)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


shapes = {"qkv": (1024, 6144, 4096, 0), "o": (1024, 4096, 4096, 0), "gate_up": (1024, 28672, 4096, 3),
          "down": (1024, 4096, 14336, 0)}
for name, (M, N, K, e) in shapes.items():
    fl = 2 * M * N * K
    row = {tile: t_gemm(M, N, K, e, tile) for tile in (0, 128, 256, 512, 640)}
    cb = t_cublas(M, N, K)
    print(f"{name:8s} M={M} N={N} K={K}: " + "  ".join(f"{k}:{v:6.1f}us({fl / v / 1e6:5.0f})" for k, v in row.items())
          + f"  cublas:{cb:6.1f}us({fl / cb / 1e6:5.0f} TF/s)", flush=True)
for name, (M, N, K, e) in shapes.items():
    row = {tile: t_gemm(M, N, K, e, tile, cold=True) for tile in (0, 256, 512, 640)}
    print(f"{name:8s} cold L2: " + "  ".join(f"{k}:{v:6.1f}us" for k, v in row.items()), flush=True)
for N in (4096, 6144):
    for K in (512, 1024, 2048, 4096, 8192):
        fl = 2 * 1024 * N * K
        row = {tile: t_gemm(1024, N, K, 0, tile) for tile in (0, 256, 512, 640)}
        print(f"sweep M=1024 N={N} K={K}: " + "  ".join(f"{k}:{v:6.1f}us" for k, v in row.items()), flush=True)
