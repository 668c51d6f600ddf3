// H1 on the GPU: the .rdkv payload checksum, 64-bit FNV-1a (codec.py:64-69),
// computed in parallel — bit-exact with the serial definition.
//
// FNV-1a is h <- (h ^ b) * P (mod 2^64), a serial chain that a CPU core walks at
// ~0.6 GB/s (140 ms for one 80 MiB C2 composite, 1.1 s for a C3 one).  It
// decomposes because the XOR only touches the low byte:
//   * the low byte s of h evolves on its own: s <- ((s ^ b) * P) mod 256, a
//     256-state automaton (P mod 256 = 0xB3; bits above 8 never flow down);
//   * given the low-byte sequence, (h ^ b) = h + d with d = (s ^ b) - s, so
//     h <- (h + d) * P is affine in h: a chunk of L bytes maps h to
//     h * P^L + C_chunk, and affine maps compose.
// Three passes:
//   1. fnv_fsm_kernel: per 16-KiB chunk, one warp runs the automaton from every
//      possible start byte (8 per lane, packed two per register; the chunk is
//      staged once in smem and read as a broadcast) -> end_state[chunk][start].
//   2. fnv_stitch_kernel: one block walks the chunks from the seed's low byte,
//      64 table rows per smem batch -> start_state[chunk].
//   3. fnv_affine_kernel: one thread per chunk runs the exact byte recurrence
//      for C_chunk from its start byte; fnv_combine_kernel folds
//      h = h * P^L + C over the chunks in order.
// ~2 ms for 80 MiB on a B200 (HBM-resident payload), vs 90-140 ms on one core.
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"
#include "pdl.cuh"

namespace rdkv {
namespace {

constexpr uint64_t kP = 0x100000001B3ull;
constexpr uint32_t kPlo = 0xB3u;
constexpr int kChunk = 16384;      // bytes per chunk (multiple of 16)
constexpr int kStage = 4096;       // smem staging bytes per pass in the automaton kernel
constexpr int kRows = 64;          // end-state rows per smem batch in the stitch kernel

__device__ __forceinline__ uint64_t pow_p(uint64_t e) {
  uint64_t r = 1, b = kP;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

// One warp per chunk; lane l runs start bytes 8l .. 8l+7 as four packed pairs
// (two 8-bit states in the low bytes of the 16-bit halves of a register): per
// input byte one PRMT replicates it into both halves, then per pair one LOP3
// ((p ^ bb) & 0x00FF00FF) and one IMAD (* 0xB3, < 2^16 so the halves never mix).
constexpr int kWarpsPerBlock = 4;
__global__ void __launch_bounds__(32 * kWarpsPerBlock) fnv_fsm_kernel(const uint8_t* __restrict__ data, size_t n,
                                                                      int c0, int chunks, uint8_t* __restrict__ end_state) {
  pdl_trigger();
  pdl_wait();
  __shared__ __align__(16) uint32_t buf[kWarpsPerBlock][kStage / 4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = c0 + blockIdx.x * kWarpsPerBlock + warp;  // chunks [c0, chunks)
  if (c >= chunks) return;
  const size_t base = (size_t)c * kChunk;
  const int len = (int)min((size_t)kChunk, n - base);
  uint32_t* wb = buf[warp];
  uint32_t p[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j] = ((uint32_t)(8 * lane + 2 * j + 1) << 16) | (uint32_t)(8 * lane + 2 * j);
  const bool aligned = ((reinterpret_cast<uintptr_t>(data) | base) & 15) == 0;
  for (int off = 0; off < len; off += kStage) {
    const int m = min(kStage, len - off);
    __syncwarp();
    if (aligned && (m & 15) == 0) {
      for (int i = lane; i < m / 16; i += 32)
        reinterpret_cast<uint4*>(wb)[i] = reinterpret_cast<const uint4*>(data + base + off)[i];
    } else {
      for (int i = lane; i < m; i += 32) reinterpret_cast<uint8_t*>(wb)[i] = data[base + off + i];
    }
    __syncwarp();
    auto step = [&](uint32_t bb) {
#pragma unroll
      for (int j = 0; j < 4; ++j) p[j] = ((p[j] ^ bb) & 0x00FF00FFu) * kPlo;
    };
    const int words = m / 4;
#pragma unroll 2
    for (int w = 0; w < words; ++w) {
      const uint32_t x = wb[w];  // same address in every lane: a broadcast
      step(__byte_perm(x, 0, 0x4040));
      step(__byte_perm(x, 0, 0x4141));
      step(__byte_perm(x, 0, 0x4242));
      step(__byte_perm(x, 0, 0x4343));
    }
    for (int i = words * 4; i < m; ++i) {
      const uint32_t v = reinterpret_cast<const uint8_t*>(wb)[i];
      step(v | (v << 16));
    }
  }
  uint8_t* row = end_state + (size_t)c * 256 + 8 * lane;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    row[2 * j] = (uint8_t)(p[j] & 0xFF);
    row[2 * j + 1] = (uint8_t)((p[j] >> 16) & 0xFF);
  }
}

__global__ void __launch_bounds__(256) fnv_stitch_kernel(const uint8_t* __restrict__ end_state, int chunks,
                                                         uint64_t seed, uint8_t* __restrict__ start_state) {
  pdl_trigger();
  pdl_wait();
  __shared__ __align__(16) uint8_t rows[kRows * 256];
  uint32_t s = (uint32_t)(seed & 0xFF);
  for (int c0 = 0; c0 < chunks; c0 += kRows) {
    const int nr = min(kRows, chunks - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < nr * 16; i += 256)
      reinterpret_cast<uint4*>(rows)[i] = reinterpret_cast<const uint4*>(end_state + (size_t)c0 * 256)[i];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int r = 0; r < nr; ++r) {
        start_state[c0 + r] = (uint8_t)s;
        s = rows[r * 256 + s];
      }
  }
}

__global__ void __launch_bounds__(128) fnv_affine_kernel(const uint8_t* __restrict__ data, size_t n, int chunks,
                                                         const uint8_t* __restrict__ start_state,
                                                         uint64_t* __restrict__ cterm) {
  pdl_trigger();
  pdl_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= chunks) return;
  const size_t base = (size_t)c * kChunk;
  const int len = (int)min((size_t)kChunk, n - base);
  uint32_t s = start_state[c];
  uint64_t C = 0;
  auto step = [&](uint32_t b) {
    const uint32_t x = (s ^ b) & 0xFF;
    C = (C + (uint64_t)((int64_t)x - (int64_t)s)) * kP;  // d = (s ^ b) - s, exact mod 2^64
    s = (x * kPlo) & 0xFF;
  };
  int i = 0;
  if (((reinterpret_cast<uintptr_t>(data) | base) & 15) == 0) {
    for (; i + 16 <= len; i += 16) {
      const uint4 v = *reinterpret_cast<const uint4*>(data + base + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        step(w[k] & 0xFF);
        step((w[k] >> 8) & 0xFF);
        step((w[k] >> 16) & 0xFF);
        step(w[k] >> 24);
      }
    }
  }
  for (; i < len; ++i) step(data[base + i]);
  cterm[c] = C;
}

// h = ((seed * A_0 + C_0) * A_1 + C_1) ...: each lane folds a contiguous run of
// chunks into one affine map (A, C), then lane 0 folds the 32 maps in order.
__global__ void fnv_combine_kernel(const uint64_t* __restrict__ cterm, int chunks, size_t n, uint64_t seed,
                                   uint64_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x;
  const uint64_t a_full = pow_p(kChunk);
  const int per = (chunks + 31) / 32;
  const int c0 = min(chunks, lane * per), c1 = min(chunks, c0 + per);
  uint64_t A = 1, C = 0;
  for (int c = c0; c < c1; ++c) {
    const size_t len = min((size_t)kChunk, n - (size_t)c * kChunk);
    const uint64_t a = len == (size_t)kChunk ? a_full : pow_p(len);
    A *= a;
    C = C * a + cterm[c];
  }
  uint64_t h = seed;
  for (int l = 0; l < 32; ++l) {
    const uint64_t Al = __shfl_sync(0xffffffffu, A, l), Cl = __shfl_sync(0xffffffffu, C, l);
    h = h * Al + Cl;
  }
  if (lane == 0) *out = h;
}

}  // namespace
}  // namespace rdkv

using namespace rdkv;

extern "C" size_t rdkv_fnv1a64_device_scratch(size_t len) {
  const size_t chunks = (len + kChunk - 1) / kChunk;
  return chunks * 256 + chunks + chunks * 8 + 64;
}

namespace {
int check_args(const void* data, size_t len, const void* scratch, size_t scratch_bytes) {
  if (len && !data) return set_error(RDKV_ERR_ARG, "fnv_device: null argument");
  const size_t chunks = (len + kChunk - 1) / kChunk;
  if (chunks > (size_t)1 << 30) return set_error(RDKV_ERR_ARG, "fnv_device: input too large");
  if (scratch_bytes < rdkv_fnv1a64_device_scratch(len) || (chunks && !scratch))
    return set_error(RDKV_ERR_ARG, "fnv_device: scratch too small");
  return 0;
}
}  // namespace

// Pass 1 alone for the whole 16-KiB chunks of bytes [0, ready) of a `len`-byte
// input, from chunk `chunk_begin` on (a payload still arriving: run it per landed
// segment, then rdkv_fnv1a64_device_finish).  Returns the next chunk to run.
extern "C" int64_t rdkv_fnv1a64_device_partial(const void* data, size_t len, size_t ready, int64_t chunk_begin,
                                               void* scratch, size_t scratch_bytes, void* stream) {
  RDKV_TRY(check_args(data, len, scratch, scratch_bytes));
  const size_t chunks = (len + kChunk - 1) / kChunk;
  const int64_t c1 = ready >= len ? (int64_t)chunks : (int64_t)(ready / kChunk);
  if (chunk_begin < 0 || chunk_begin > c1) return set_error(RDKV_ERR_ARG, "fnv_device: bad chunk range");
  if (c1 > chunk_begin) {
    const int n = (int)(c1 - chunk_begin);
    CUDA_TRY(launch_k(fnv_fsm_kernel, dim3((n + kWarpsPerBlock - 1) / kWarpsPerBlock), dim3(32 * kWarpsPerBlock), 0,
                      static_cast<cudaStream_t>(stream), static_cast<const uint8_t*>(data), len, (int)chunk_begin,
                      (int)c1, static_cast<uint8_t*>(scratch)));
    CUDA_TRY(cudaGetLastError());
  }
  return c1;
}

// Passes 2-4 (after pass 1 covered every chunk): *out_dev on `stream`.
extern "C" int rdkv_fnv1a64_device_finish(const void* data, size_t len, uint64_t seed, void* scratch,
                                          size_t scratch_bytes, uint64_t* out_dev, void* stream) {
  if (!out_dev) return set_error(RDKV_ERR_ARG, "fnv_device: null argument");
  RDKV_TRY(check_args(data, len, scratch, scratch_bytes));
  const size_t chunks = (len + kChunk - 1) / kChunk;
  auto st = static_cast<cudaStream_t>(stream);
  auto* ws = static_cast<uint8_t*>(scratch);
  uint8_t* end_state = ws;                                   // [chunks][256]
  uint64_t* cterm = reinterpret_cast<uint64_t*>(ws + ((chunks * 256 + 7) / 8) * 8);  // [chunks]
  uint8_t* start_state = reinterpret_cast<uint8_t*>(cterm + chunks);                   // [chunks]
  const auto* d = static_cast<const uint8_t*>(data);
  const int nc = (int)chunks;
  if (nc > 0) {
    CUDA_TRY(launch_k(fnv_stitch_kernel, dim3(1), dim3(256), 0, st, (const uint8_t*)end_state, nc, seed, start_state));
    CUDA_TRY(launch_k(fnv_affine_kernel, dim3((nc + 127) / 128), dim3(128), 0, st, d, len, nc,
                      (const uint8_t*)start_state, cterm));
  }
  CUDA_TRY(launch_k(fnv_combine_kernel, dim3(1), dim3(32), 0, st, (const uint64_t*)cterm, nc, len, seed, out_dev));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Device FNV-1a of `len` bytes at `data` (device memory), written to
// *out_dev (device uint64) asynchronously on `stream`.
extern "C" int rdkv_fnv1a64_device(const void* data, size_t len, uint64_t seed, void* scratch, size_t scratch_bytes,
                                   uint64_t* out_dev, void* stream) {
  if (!out_dev) return set_error(RDKV_ERR_ARG, "fnv_device: null argument");
  const int64_t c = rdkv_fnv1a64_device_partial(data, len, len, 0, scratch, scratch_bytes, stream);
  if (c < 0) return (int)c;
  return rdkv_fnv1a64_device_finish(data, len, seed, scratch, scratch_bytes, out_dev, stream);
}
