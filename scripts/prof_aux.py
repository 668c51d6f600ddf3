"""Dev: one launch each of the auxiliary hot-path kernels for ncu captures —
GPU FNV-1a of an 80 MiB payload, K3 unpack of 32 C2 composites, K3p block gather
(same-GPU source), and the TP reduce kernel is covered by the TP tests."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_11765_b200 import codec
from paper_2504_11765_b200.engine import Engine, KvPool, kv_unpack, pack_unpack_jobs
from paper_2504_11765_b200.model import get_spec
from paper_2504_11765_b200 import _lib
from paper_2504_11765_b200.engine import _L

spec = get_spec("llama-3.2-1b")
x = torch.randint(0, 256, (80 << 20,), dtype=torch.uint8, device="cuda")
codec.fnv1a64_device(x)
n, B = 2560, 32
pool = KvPool(spec, n_blocks=2 * B * (n // 64) + 8, block_size=64)
payloads = [torch.randn(spec.layers * 2 * spec.kv_heads * n * spec.head_dim, device="cuda").bfloat16() for _ in range(B)]
blocks = pool.alloc_blocks(B * n // 64)
bt = torch.tensor(blocks, dtype=torch.int32, device="cuda")
jobs = [(p, n, i * (n // 64)) for i, p in enumerate(payloads)]
kv_unpack(pool, jobs, bt, jobs_dev=pack_unpack_jobs(jobs).to("cuda"))
dst = pool.alloc_blocks(len(blocks))
s = torch.tensor(blocks, dtype=torch.int32, device="cuda")
d = torch.tensor(dst, dtype=torch.int32, device="cuda")
_lib.check(_L().rdkv_kv_peer_gather(pool.data.data_ptr(), pool.slots, s.data_ptr(), pool.data.data_ptr(), pool.slots,
                                    d.data_ptr(), len(blocks), spec.layers, spec.kv_heads, spec.head_dim, 64,
                                    torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("done")
