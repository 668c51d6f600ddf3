"""K1 tcgen05 GEMM parity against a plain PyTorch fp32 reference of the same op,
for both tile widths (N=128, N=256), every exposed epilogue, and the split-K
path small-M shapes take (fp32 partial slabs + fixed-order finalize)."""

import pytest
import torch

from paper_2504_11765_b200 import _lib

pytestmark = pytest.mark.gpu

TILES = [0, 128, 256, 384, 512, 640]  # 0 automatic; 384 / 512 / 640 = CTA-pair (cta_group::2) 256x128 / 256x256 / 256x384 tiles


def _ptr(t):
    return t.data_ptr() if t is not None else None


def _gemm(A, B, D, epi, R=None, tile=0, scratch=None):
    s = torch.cuda.current_stream().cuda_stream
    M, K = A.shape
    if tile in (384, 512, 640) and M < 256:
        pytest.skip("CTA-pair tiles need M >= 256")
    N = B.shape[0]
    if tile == 640 and N % 384:
        pytest.skip("256x384 tiles need N % 384 == 0")
    _lib.check(_lib.lib().rdkv_gemm_bf16_ex(
        _ptr(A), A.stride(0), _ptr(B), B.stride(0), _ptr(D), D.stride(0),
        _ptr(R), R.stride(0) if R is not None else 0, M, N, K, epi, tile,
        _ptr(scratch), scratch.numel() if scratch is not None else 0, s))


def _inputs(M, N, K, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = (torch.randn(M, K, device="cuda", generator=g) / K ** 0.25).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.25).to(torch.bfloat16)
    return A, B


SHAPES = [(128, 128, 64), (256, 384, 512), (200, 96, 128), (37, 4096, 2048), (2048, 2048, 2048),
          (1000, 3072, 2048), (2048, 3072, 2048), (64, 2048, 8192)]  # N = 3072: 256 x 192 CTA-pair tiles
SCRATCH = 64 << 20  # bytes: enables split-K for the small-M shapes below


@pytest.fixture(scope="module")
def scratch():
    return torch.empty(SCRATCH, dtype=torch.uint8, device="cuda")


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("tile", TILES)
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_store_bf16(M, N, K, tile, split, scratch):
    A, B = _inputs(M, N, K)
    D = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    _gemm(A, B, D, _lib.EPI_STORE, tile=tile, scratch=scratch if split else None)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    torch.testing.assert_close(D.float(), ref, atol=2e-2, rtol=1e-2)


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("tile", TILES)
@pytest.mark.parametrize("M,N,K", [(33, 1024, 256), (128, 128256 // 4, 2048), (8, 2048, 2048)])
def test_store_f32(M, N, K, tile, split, scratch):
    A, B = _inputs(M, N, K, seed=1)
    D = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    _gemm(A, B, D, _lib.EPI_STORE_F32, tile=tile, scratch=scratch if split else None)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    torch.testing.assert_close(D, ref, atol=1e-3, rtol=1e-3)


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("tile", TILES)
@pytest.mark.parametrize("M,N,K", [(300, 512, 1024), (2048, 2048, 8192), (64, 2048, 8192), (512, 3072, 1024)])
def test_residual_in_place(M, N, K, tile, split, scratch):
    A, B = _inputs(M, N, K, seed=2)
    X = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    ref = X.float() + A.float() @ B.float().T
    _gemm(A, B, X, _lib.EPI_RESID, tile=tile, scratch=scratch if split else None)
    torch.cuda.synchronize()
    torch.testing.assert_close(X.float(), ref, atol=3e-2, rtol=1e-2)


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("tile", TILES)
@pytest.mark.parametrize("M,N,K", [(130, 256, 128), (640, 2 * 8192, 2048), (64, 384, 512), (64, 4096, 2048), (512, 3072, 512)])
def test_swiglu(M, N, K, tile, split, scratch):
    A, B = _inputs(M, N, K, seed=3)
    D = torch.full((M, N // 2), float("nan"), device="cuda", dtype=torch.bfloat16)
    _gemm(A, B, D, _lib.EPI_SWIGLU, tile=tile, scratch=scratch if split else None)
    torch.cuda.synchronize()
    full = (A.float() @ B.float().T).view(M, N // 128, 2, 64)
    ref = (torch.nn.functional.silu(full[:, :, 0]) * full[:, :, 1]).reshape(M, N // 2)
    torch.testing.assert_close(D.float(), ref, atol=2e-2, rtol=1e-2)


def test_split_k_is_deterministic(scratch):
    A, B = _inputs(64, 2048, 8192, seed=4)
    outs = []
    for _ in range(3):
        D = torch.empty(64, 2048, device="cuda", dtype=torch.bfloat16)
        _gemm(A, B, D, _lib.EPI_STORE, scratch=scratch)
        outs.append(D)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


def test_bad_k_rejected():
    A, B = _inputs(128, 128, 96)
    D = torch.empty(128, 128, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(_lib.NativeError):
        _gemm(A, B, D, _lib.EPI_STORE)


@pytest.mark.parametrize("epi", [_lib.EPI_STORE, _lib.EPI_SWIGLU])
def test_last_round_tail_tiles(epi):
    """M = 1024, N = 28672 (the C3 gate/up shape): 448 tiles of 256 x 256 on 74 CTA pairs
    leave a 7th round of 4 tiles (with RDKV_GEMM_TAIL=1 the last 256 columns run as a second
    launch of 256 x 128 tiles).  Every column, the last tile column included, matches."""
    M, N, K = 1024, 28672, 256
    A, B = _inputs(M, N, K, seed=5)
    n_out = N // 2 if epi == _lib.EPI_SWIGLU else N
    D = torch.full((M, n_out), float("nan"), device="cuda", dtype=torch.bfloat16)
    _gemm(A, B, D, epi)
    torch.cuda.synchronize()
    full = A.float() @ B.float().T
    if epi == _lib.EPI_SWIGLU:
        f = full.view(M, N // 128, 2, 64)
        ref = (torch.nn.functional.silu(f[:, :, 0]) * f[:, :, 1]).reshape(M, n_out)
    else:
        ref = full
    torch.testing.assert_close(D.float(), ref, atol=2e-2, rtol=1e-2)
