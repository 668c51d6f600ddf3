"""Dev microbenchmark: K1 GEMM TFLOP/s vs torch (cuBLAS) on the model's shapes."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_11765_b200 import _lib

def run(M, N, K, epi=_lib.EPI_STORE, iters=20):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    n_out = N // 2 if epi == _lib.EPI_SWIGLU else N
    D = torch.empty(M, n_out, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    L = _lib.lib()
    f = lambda: L.rdkv_gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, D.data_ptr(), n_out, None, 0, M, N, K, epi, s)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): f()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / iters
    for _ in range(3): torch.matmul(A, B.T)
    e0.record()
    for _ in range(iters): torch.matmul(A, B.T)
    e1.record(); torch.cuda.synchronize()
    tc = e0.elapsed_time(e1) / iters
    fl = 2 * M * N * K
    print(f"M={M:6d} N={N:6d} K={K:6d} epi={epi}: rdkv {t*1e3:8.1f} us {fl/t/1e9:7.1f} TF/s | cublas {tc*1e3:8.1f} us {fl/tc/1e9:7.1f} TF/s", flush=True)

for (M, N, K, e) in [(8192, 8192, 8192, 0), (4096, 4096, 4096, 0), (2560, 3072, 2048, 0), (2560, 16384, 2048, 3),
                     (2560, 2048, 8192, 0), (5120, 6144, 4096, 0), (5120, 28672, 4096, 3), (5120, 4096, 14336, 0),
                     (2048, 2048, 2048, 0), (640, 2048, 2048, 0), (64, 16384, 2048, 3), (32, 128256, 2048, 0)]:
    run(M, N, K, e)
