"""One GEMM shape through the C ABI, launched a few times (for ncu metric captures):
    python scripts/gemm_one.py M N K [epi] [tile]   (epi: store | swiglu; tile 0 = planner)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2504_11765_b200 import _lib

M, N, K = (int(x) for x in sys.argv[1:4])
epi = _lib.EPI_SWIGLU if len(sys.argv) > 4 and sys.argv[4] == "swiglu" else _lib.EPI_STORE
tile = int(sys.argv[5]) if len(sys.argv) > 5 else 0
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
n_out = N // 2 if epi == _lib.EPI_SWIGLU else N
D = torch.empty(M, n_out, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream
L = _lib.lib()
for _ in range(4):
    _lib.check(L.rdkv_gemm_bf16_ex(A.data_ptr(), K, B.data_ptr(), K, D.data_ptr(), n_out, None, 0, M, N, K, epi,
                                   tile, None, 0, s))
torch.cuda.synchronize()
