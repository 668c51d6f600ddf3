"""Dev: time each K1 tile configuration (tile_n 128/256 single CTA, 384/512 CTA pairs)
on given shapes, to calibrate the planner (gemm_tc.cu pick_tiles)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_11765_b200 import _lib


def t_gemm(M, N, K, epi, tile, iters=20):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    n_out = N // 2 if epi == _lib.EPI_SWIGLU else N
    D = torch.empty(M, n_out, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    L = _lib.lib()
    f = lambda: _lib.check(L.rdkv_gemm_bf16_ex(A.data_ptr(), K, B.data_ptr(), K, D.data_ptr(), n_out, None, 0, M, N, K,
                                               epi, tile, None, 0, s))
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


shapes = [(2048, 3072, 2048, 0), (2048, 2048, 2048, 0), (2048, 16384, 2048, 3), (2048, 2048, 8192, 0),
          (4096, 3072, 2048, 0), (1024, 3072, 2048, 0), (2368, 3072, 2048, 0)]
for M, N, K, e in shapes:
    row = {tile: t_gemm(M, N, K, e, tile) for tile in (0, 128, 256, 384, 512)}
    print(f"M={M} N={N} K={K} epi={e}: " + "  ".join(f"{k}:{v:6.1f}us" for k, v in row.items()), flush=True)
