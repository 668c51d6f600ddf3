"""Small-M (decode / single-query) K1 GEMMs at the Llama-3-8B shapes: swap-AB split-K +
finalize through rdkv_gemm_bf16_ex, cold weights (a >L2 buffer written between launches),
as GB/s of weight bytes against the HBM copy peak; cuBLAS (torch.matmul) beside it.

    python scripts/gemm_small_m.py [M ...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2504_11765_b200 import _lib

FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
SHAPES = {"qkv": (6144, 4096, 0), "o": (4096, 4096, 2), "gate_up": (28672, 4096, 3), "down": (4096, 14336, 2)}


def timed(f, iters=20):
    evs = []
    for _ in range(iters):
        FLUSH.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in evs)[iters // 2] * 1e3  # median us


def main():
    Ms = [int(x) for x in sys.argv[1:]] or [16, 64]
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for M in Ms:
        for name, (N, K, e) in SHAPES.items():
            A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
            n_out = N // 2 if e == 3 else N
            D = torch.empty(M, n_out, device="cuda", dtype=torch.bfloat16)
            R = torch.randn(M, n_out, device="cuda").to(torch.bfloat16)
            f = lambda: _lib.check(L.rdkv_gemm_bf16_ex(A.data_ptr(), K, B.data_ptr(), K, D.data_ptr(), n_out,
                                                       R.data_ptr() if e == 2 else None, n_out, M, N, K, e, 0,
                                                       ws.data_ptr(), ws.numel(), s))
            for _ in range(3):
                f()
            t = timed(f)
            tc = timed(lambda: torch.matmul(A, B.T))
            gb = N * K * 2 / 1e9
            print(f"M={M:3d} {name:8s} N={N:6d} K={K:6d}: rdkv {t:6.1f} us {gb / t * 1e6:7.0f} GB/s | "
                  f"cublas {tc:6.1f} us {gb / tc * 1e6:7.0f} GB/s", flush=True)


main()
