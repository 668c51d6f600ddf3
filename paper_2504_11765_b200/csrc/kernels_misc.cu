// HBM-bound helper kernels of the hot path:
//   K3  kv_unpack     blob payload [L][2][Hkv][n][dh] (bf16 or fp32) -> paged pool planes
//       embed         token ids -> residual rows
//       rmsnorm       row RMSNorm with fp32 gain (optionally gathering rows)
//       argmax        first index of the row maximum (torch.argmax tie rule)
#include <cuda_bf16.h>
#include <cstdint>

#include "common.cuh"
#include "kernels_misc.cuh"
#include "pdl.cuh"

namespace rdkv {
namespace {

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---------------------------------------------------------------- K3 unpack
// One warp moves one segment = (job, layer, k|v, head, block): a contiguous
// run of up to block_size*dh elements in the blob and in the pool plane.
// 16-byte loads, UNROLL of them in flight per lane.
// Heads [h0, h0 + hkv) of a payload holding src_hkv heads land in a pool of hkv
// heads (a tensor-parallel rank reads its own heads of a full-model blob: each
// is a contiguous [n][dh] run of the head-major payload).
template <int SRC_W>
__global__ void __launch_bounds__(256) kv_unpack_kernel(const UnpackJob* __restrict__ jobs, const int* __restrict__ bt,
                                                        int block_size, __nv_bfloat16* __restrict__ pool, int layer0,
                                                        int layers, int hkv, int dh, long long slots, int h0,
                                                        int src_hkv) {
  pdl_trigger();
  pdl_wait();
  const UnpackJob jb = jobs[blockIdx.y];
  const int nblk = (jb.n_tokens + block_size - 1) / block_size;
  const long long nseg = (long long)layers * 2 * hkv * nblk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int UNROLL = 4;
  for (long long seg = (long long)blockIdx.x * 8 + warp; seg < nseg; seg += (long long)gridDim.x * 8) {
    const int b = (int)(seg % nblk);
    const int plane = layer0 * 2 * hkv + (int)(seg / nblk);  // (l*2 + kv)*hkv + h  (< 2^31)
    const int src_plane = src_hkv == hkv ? plane : (plane / hkv) * src_hkv + h0 + plane % hkv;
    const int t0 = b * block_size;
    const int ntok = min(block_size, jb.n_tokens - t0);
    const long long n_el = (long long)ntok * dh;
    const long long src_off = (long long)src_plane * jb.n_tokens * dh + (long long)t0 * dh;
    const long long dst_off = (long long)plane * slots * dh + (long long)bt[jb.first_block + b] * block_size * dh;
    __nv_bfloat16* dst = pool + dst_off;
    if constexpr (SRC_W == 2) {
      const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(jb.src) + src_off;
      const long long nvec = n_el / 8;  // 8 bf16 per 16 B
      long long i = lane;
      for (; i + 32 * (UNROLL - 1) < nvec; i += 32 * UNROLL) {
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = ld_stream(src + (i + 32 * u) * 8);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) *reinterpret_cast<uint4*>(dst + (i + 32 * u) * 8) = v[u];
      }
      for (; i < nvec; i += 32) *reinterpret_cast<uint4*>(dst + i * 8) = ld_stream(src + i * 8);
    } else {
      const float* src = static_cast<const float*>(jb.src) + src_off;
      const long long nvec = n_el / 8;  // 8 fp32 (32 B) -> 8 bf16 (16 B)
      for (long long i = lane; i < nvec; i += 32) {
        const uint4 a = ld_stream(src + i * 8), c = ld_stream(src + i * 8 + 4);
        uint4 o;
        o.x = pack_bf16_f(__uint_as_float(a.x), __uint_as_float(a.y));
        o.y = pack_bf16_f(__uint_as_float(a.z), __uint_as_float(a.w));
        o.z = pack_bf16_f(__uint_as_float(c.x), __uint_as_float(c.y));
        o.w = pack_bf16_f(__uint_as_float(c.z), __uint_as_float(c.w));
        *reinterpret_cast<uint4*>(dst + i * 8) = o;
      }
    }
  }
}

// ---------------------------------------------------------------- embed
// With ssq != null also the first RMSNorm's statistics: per row and 32-column chunk
// the sum of squares, ssq[chunk][n] (the layout GEMM residual epilogues write).
__global__ void embed_kernel(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ table,
                             __nv_bfloat16* __restrict__ out, int d, int vocab, float* __restrict__ ssq, int n) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  int id = tok[t];
  id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);
  const uint4* src = reinterpret_cast<const uint4*>(table + (long long)id * d);
  uint4* dst = reinterpret_cast<uint4*>(out + (long long)t * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {  // blockDim is a multiple of 4: chunks stay in-warp
    const uint4 v = src[i];
    dst[i] = v;
    if (ssq) {
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = unpack_bf16_f(w[j]);
        ss = fmaf(f.x, f.x, ss);
        ss = fmaf(f.y, f.y, ss);
      }
      ss += __shfl_xor_sync(0xffffffff, ss, 1);
      ss += __shfl_xor_sync(0xffffffff, ss, 2);
      if ((i & 3) == 0) ssq[(long long)(i >> 2) * n + t] = ss;
    }
  }
}

// ---------------------------------------------------------------- rmsnorm
// out[r] = x[src_row(r)] * rsqrt(mean(x^2) + eps) * gain.
// Warp per row, the row held in registers (CH 16-byte chunks per lane, d <=
// 256*CH), so x is read once: one HBM pass in, one out.
template <int CH>
__global__ void __launch_bounds__(256) rmsnorm_warp_kernel(const __nv_bfloat16* __restrict__ x, long long ldx,
                                                           const int* __restrict__ rows,
                                                           const float* __restrict__ gain,
                                                           __nv_bfloat16* __restrict__ out, long long ldo, int n_rows,
                                                           int d, float eps) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + warp;
  if (r >= n_rows) return;
  const int src_row = rows ? rows[r] : r;
  const __nv_bfloat16* xr = x + (long long)src_row * ldx;
  uint4 v[CH];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int i = (c * 32 + lane) * 8;
    v[c] = i < d ? ld_stream(xr + i) : make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16_f(w[j]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  const float inv = rsqrtf(ss / (float)d + eps);
  __nv_bfloat16* orow = out + (long long)r * ldo;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int i = (c * 32 + lane) * 8;
    if (i >= d) break;
    const float4 g0 = *reinterpret_cast<const float4*>(gain + i);
    const float4 g1 = *reinterpret_cast<const float4*>(gain + i + 4);
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const uint32_t w[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = unpack_bf16_f(w[j]);
      o[j] = pack_bf16_f(f.x * inv * gg[2 * j], f.y * inv * gg[2 * j + 1]);
    }
    *reinterpret_cast<uint4*>(orow + i) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ---------------------------------------------------------------- argmax
// Two stages so a [rows x 128k] logit matrix spreads over many SMs:
// (1) grid (rows, ARGMAX_CH): each CTA reduces a contiguous chunk -> (value, index);
// (2) one warp per row reduces the chunk winners.  Ties resolve to the lowest
// index (torch.argmax's first-occurrence rule) at every level.
constexpr int ARGMAX_CH = 32;

__device__ __forceinline__ void argmax_merge(float& best, int& idx, float vb, int ib) {
  if (vb > best || (vb == best && ib < idx)) {
    best = vb;
    idx = ib;
  }
}

__global__ void __launch_bounds__(256) argmax_chunk_kernel(const float* __restrict__ logits, long long ld, int n,
                                                          float2* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x, ch = blockIdx.y;
  const int len = (n + ARGMAX_CH - 1) / ARGMAX_CH;
  const int lo = ch * len, hi = min(n, lo + len);
  const float* r = logits + (long long)row * ld;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) argmax_merge(best, idx, r[i], i);
  for (int o = 16; o; o >>= 1)
    argmax_merge(best, idx, __shfl_xor_sync(0xffffffff, best, o), __shfl_xor_sync(0xffffffff, idx, o));
  __shared__ float sv[8];
  __shared__ int si[8];
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < 8 ? sv[threadIdx.x] : -INFINITY;
    idx = threadIdx.x < 8 ? si[threadIdx.x] : 0x7fffffff;
    for (int o = 16; o; o >>= 1)
      argmax_merge(best, idx, __shfl_xor_sync(0xffffffff, best, o), __shfl_xor_sync(0xffffffff, idx, o));
    if (threadIdx.x == 0) part[row * ARGMAX_CH + ch] = make_float2(best, __int_as_float(idx));
  }
}

__global__ void argmax_final_kernel(const float2* __restrict__ part, int* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x, lane = threadIdx.x;
  const float2 p = part[row * ARGMAX_CH + lane];
  float best = p.x;
  int idx = __float_as_int(p.y);
  for (int o = 16; o; o >>= 1)
    argmax_merge(best, idx, __shfl_xor_sync(0xffffffff, best, o), __shfl_xor_sync(0xffffffff, idx, o));
  if (lane == 0) out[row] = idx;
}

}  // namespace

int launch_kv_unpack(const UnpackJob* jobs_dev, int n_jobs, int max_tokens, const int* bt, int block_size,
                     void* pool, int layer_begin, int layer_end, int hkv, int dh, long long slots, int elem_width,
                     cudaStream_t st, int head_begin, int src_kv_heads) {
  const int layers = layer_end - layer_begin;
  if (n_jobs <= 0 || max_tokens <= 0 || layers <= 0) return 0;
  if (dh % 8 != 0) return set_error(RDKV_ERR_ARG, "unpack: head_dim must be a multiple of 8");
  if (elem_width != 2 && elem_width != 4) return set_error(RDKV_ERR_ARG, "unpack: elem_width must be 2 or 4");
  if (src_kv_heads <= 0) src_kv_heads = hkv;
  if (head_begin < 0 || head_begin + hkv > src_kv_heads)
    return set_error(RDKV_ERR_ARG, "unpack: heads [%d, %d) outside the payload's %d", head_begin, head_begin + hkv,
                     src_kv_heads);
  const long long segs = (long long)layers * 2 * hkv * ((max_tokens + block_size - 1) / block_size);
  long long gx = (segs + 7) / 8;
  const long long cap = 4LL * num_sms() * 4;  // ~4 CTAs/SM resident, a few waves
  if (gx > cap) gx = cap;
  dim3 grid((unsigned)gx, (unsigned)n_jobs);
  auto* dst = static_cast<__nv_bfloat16*>(pool);
  if (elem_width == 2)
    CUDA_TRY(launch_k(kv_unpack_kernel<2>, grid, dim3(256), 0, st, jobs_dev, bt, block_size, dst, layer_begin, layers,
                      hkv, dh, slots, head_begin, src_kv_heads));
  else
    CUDA_TRY(launch_k(kv_unpack_kernel<4>, grid, dim3(256), 0, st, jobs_dev, bt, block_size, dst, layer_begin, layers,
                      hkv, dh, slots, head_begin, src_kv_heads));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int launch_embed(const int* tok, const __nv_bfloat16* table, __nv_bfloat16* out, int n, int d, int vocab,
                 cudaStream_t st, float* ssq) {
  if (n <= 0) return 0;
  if (ssq && d % 256 != 0) return set_error(RDKV_ERR_ARG, "embed: fused norm statistics need d %% 256 == 0");
  CUDA_TRY(launch_k(embed_kernel, dim3(n), dim3(128), 0, st, tok, table, out, d, vocab, ssq, n));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int launch_rmsnorm(const __nv_bfloat16* x, long long ldx, const int* rows, const float* gain, __nv_bfloat16* out,
                   long long ldo, int n_rows, int d, float eps, cudaStream_t st) {
  if (n_rows <= 0) return 0;
  if (d % 8 != 0 || d > 8192) return set_error(RDKV_ERR_ARG, "rmsnorm: d must be a multiple of 8 and <= 8192");
  const dim3 grid((n_rows + 7) / 8), block(256);
  if (d <= 2048)
    CUDA_TRY(launch_k(rmsnorm_warp_kernel<8>, grid, block, 0, st, x, ldx, rows, gain, out, ldo, n_rows, d, eps));
  else if (d <= 4096)
    CUDA_TRY(launch_k(rmsnorm_warp_kernel<16>, grid, block, 0, st, x, ldx, rows, gain, out, ldo, n_rows, d, eps));
  else
    CUDA_TRY(launch_k(rmsnorm_warp_kernel<32>, grid, block, 0, st, x, ldx, rows, gain, out, ldo, n_rows, d, eps));
  return 0;
}

size_t argmax_scratch_bytes(int rows) { return (size_t)(rows > 0 ? rows : 1) * ARGMAX_CH * sizeof(float2); }

int launch_argmax(const float* logits, long long ld, int rows, int n, int* out, void* scratch, cudaStream_t st) {
  if (rows <= 0) return 0;
  static_assert(ARGMAX_CH == 32, "final stage is one warp");
  auto* part = static_cast<float2*>(scratch);
  CUDA_TRY(launch_k(argmax_chunk_kernel, dim3(rows, ARGMAX_CH), dim3(256), 0, st, logits, ld, n, part));
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(launch_k(argmax_final_kernel, dim3(rows), dim3(32), 0, st, part, out));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace rdkv
